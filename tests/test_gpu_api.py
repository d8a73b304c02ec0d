"""The reference API's behaviours, exercised on the GPU implementation.

Each test restates a case of the reference's own suite (pkg/tests/,
file:line in the docstring) against paper_2105_08764_b200, so a user of the
reference sees the same contract: known-answer dyadic vectors bit for bit,
state transitions, termination, acting, targets, replay regeneration,
training-step bookkeeping and finite-difference gradients."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2105_08764_b200 as P
from paper_2105_08764_b200.policy import PARAM_NAMES, param_shapes
from reference_math import relative_error

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
KAT = json.loads((GOLD / "kat_dyadic.json").read_text())
PATH3 = P.Graph(3, [(0, 1), (1, 2)])
CYCLE5 = P.Graph(5, [(0, 1), (1, 2), (2, 3), (3, 4), (0, 4)])
TRIANGLE = P.Graph(3, [(0, 1), (1, 2), (0, 2)])
STAR4 = P.Graph(4, [(0, 1), (0, 2), (0, 3)])


def hand_params(layers, dtype=np.float64):
    return P.PolicyParams(num_layers=layers, **{
        k: np.asarray(v, dtype=dtype) for k, v in KAT["HAND_THETA"].items()})


def zero_params(k=4, layers=2):
    shapes = param_shapes(k)
    return P.PolicyParams(num_layers=layers, **{
        n: np.zeros(shapes[n], dtype=np.float32) for n in PARAM_NAMES})


def run_forward(graph, params, p, solution=None, cand=None):
    def worker(comm):
        part = P.partition_rows(graph.num_nodes, comm.size)[comm.rank]
        sol = None
        if solution is not None:
            sol = np.zeros((1, graph.num_nodes), np.uint8)
            sol[0, list(solution)] = 1
        st = P.PartitionedState([graph], part, solutions=sol, dtype=params.dtype)
        emb = P.embed_forward(st, params, comm)
        use = st.cand
        if cand is not None:
            use = np.asarray(cand, np.uint8)[None, part.row_start:part.row_stop]
        sc = P.q_forward(emb, use, params, comm)
        return comm.all_gather(emb, axis=-1), comm.all_gather(sc, axis=-1)
    return P.run_workers(p, worker)[0]


class TestDyadicKnownAnswers:
    """pkg/tests/test_policy.py:90-136 (exact equality)."""

    @pytest.mark.parametrize("p", [1, 2])
    def test_path_layers(self, p):
        e1, _ = run_forward(PATH3, hand_params(1), p)
        assert np.array_equal(e1[0], KAT["EXPECTED_PATH_L1"])
        e2, s2 = run_forward(PATH3, hand_params(2), p, cand=[1, 1, 1])
        assert np.array_equal(e2[0], KAT["EXPECTED_PATH_L2"])
        assert np.array_equal(s2[0], KAT["EXPECTED_PATH_SCORES"])

    def test_candidate_extractor(self):
        _, s = run_forward(PATH3, hand_params(2), 1, cand=[1, 0, 1])
        assert np.array_equal(s[0], KAT["EXPECTED_PATH_SCORES_EXTRACT"])

    def test_partial_solution_cycle(self):
        e, s = run_forward(CYCLE5, hand_params(2), 1, solution={0})
        assert np.array_equal(e[0], KAT["EXPECTED_CYCLE_L2"])
        assert np.array_equal(s[0, 1:], np.asarray(KAT["EXPECTED_CYCLE_SCORES"])[1:])


class TestForwardProperties:
    """pkg/tests/test_policy.py:73-88,139-162."""

    def test_all_zero_params_give_zero_outputs(self):
        e, s = run_forward(P.generate_er(10, 0.4, 3), zero_params(4, 2), 1)
        assert not e.any() and not s.any()

    def test_isolated_node_stays_zero(self):
        e, _ = run_forward(P.Graph(4, [(1, 2), (2, 3)]), P.PolicyParams.initialize(8, 2, seed=1), 1)
        assert not e[0, :, 0].any() and e[0, :, 1:].any()

    def test_permutation_equivariance_exact(self):
        g = P.Graph(6, [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (0, 5), (1, 4)])
        perm = np.array([3, 5, 0, 1, 4, 2])
        gp = P.Graph(6, [(perm[u], perm[v]) for u, v in g.edge_array])
        eb, sb = run_forward(g, hand_params(2), 1, solution={1, 4})
        ep, sp = run_forward(gp, hand_params(2), 1, solution={int(perm[1]), int(perm[4])})
        for v in range(6):
            assert np.array_equal(eb[0][:, v], ep[0][:, perm[v]])
            assert sb[0][v] == sp[0][perm[v]]


def gather_state(state, comm):
    cand = comm.all_gather(state.cand[0], axis=-1)
    sol = comm.all_gather(state.sol[0], axis=-1)
    rows, cols = state.local_residual_coo(0)
    return cand, sol, set(zip(rows.tolist(), cols.tolist()))


class TestStateTransitions:
    """pkg/tests/test_state.py:47-133."""

    @pytest.mark.parametrize("p", [1, 2])
    def test_worked_example(self, p):
        g = P.Graph(8, [(0, 2), (2, 4), (5, 7), (1, 6), (1, 3)])
        sol = np.zeros((1, 8), np.uint8)
        sol[0, 2] = 1

        def worker(comm):
            st = P.PartitionedState([g], P.partition_rows(8, comm.size)[comm.rank], solutions=sol)
            before = gather_state(st, comm)
            st.apply_action(5, slot=0)
            return before, gather_state(st, comm)
        before, after = P.run_workers(p, worker)[0]
        assert np.flatnonzero(before[0]).tolist() == [1, 3, 5, 6, 7]
        assert np.flatnonzero(after[0]).tolist() == [1, 3, 6]
        assert np.flatnonzero(after[1]).tolist() == [2, 5]

    def test_star_center_clears_everything(self):
        def worker(comm):
            st = P.PartitionedState([STAR4], P.partition_rows(4, comm.size)[comm.rank])
            st.apply_action(0)
            return gather_state(st, comm)
        cand, sol, residual = P.run_workers(2, worker)[0]
        assert not cand.any() and sol.tolist() == [1, 0, 0, 0] and residual == set()

    def test_triangle(self):
        def worker(comm):
            st = P.PartitionedState([TRIANGLE], P.partition_rows(3, 1)[0])
            st.apply_action(0)
            out = gather_state(st, comm)
            partial = st.is_covered(0, comm)
            st.apply_action(1)
            return out, partial, st.is_covered(0, comm)
        (cand, _, residual), partial, full = P.run_workers(1, worker)[0]
        assert np.flatnonzero(cand).tolist() == [1, 2]
        assert residual == {(1, 2), (2, 1)}
        assert (partial, full) == (False, True)

    def test_rejections(self):
        def worker(comm):
            st = P.PartitionedState([STAR4], P.partition_rows(4, 1)[0])
            st.apply_action(0)
            with pytest.raises(P.InvalidActionError, match="already"):
                st.apply_action(0)
            with pytest.raises(P.InvalidActionError, match="not a candidate"):
                st.apply_action(1)
            with pytest.raises(P.InvalidActionError, match="out of range"):
                st.apply_action(9)
            return True
        assert P.run_workers(1, worker) == [True]

    def test_residual_matches_reconstruction_after_random_plays(self):
        """pkg/tests/test_state.py:135-169: after random valid plays the
        residual entries and candidates equal a from-scratch rebuild."""
        rng = np.random.default_rng(5)
        g = P.generate_ba(300, 3, 11)

        def worker(comm):
            part = P.partition_rows(300, comm.size)[comm.rank]
            st = P.PartitionedState([g], part)
            chosen = []
            for _ in range(40):
                cand = comm.all_gather(st.cand[0], axis=-1)
                idx = np.flatnonzero(cand)
                if idx.size == 0:
                    break
                v = int(idx[rng.integers(idx.size)]) if comm.rank == 0 else 0
                v = int(comm.all_reduce_sum(np.array([v]))[0])
                st.apply_action(v)
                chosen.append(v)
            sol = np.zeros((1, 300), np.uint8)
            sol[0, chosen] = 1
            fresh = P.PartitionedState([g], part, solutions=sol)
            return (gather_state(st, comm), gather_state(fresh, comm), st.local_residual.copy(),
                    fresh.local_residual.copy())
        for a, b, ra, rb in P.run_workers(2, worker):
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
            assert np.array_equal(ra, rb)


@pytest.mark.parametrize("p", [1, 2])
def test_state_build_with_long_rows(p):
    """Rows over 1,024 entries take shard_init's CTA-per-row pass: candidates,
    residual entries and per-slot residual counts equal the state.py:60-90
    definition (an entry is alive iff neither endpoint is in S) on hubs of
    3,000 and 1,500 entries in a batch of two solutions, at P = 1 and 2."""
    rng = np.random.default_rng(3)
    n = 4000
    edges = {(0, v) for v in range(1, 3001)} | {(1, v) for v in range(2000, 3500)}
    while len(edges) < 3000 + 1500 + 6000:
        a, b = sorted(rng.integers(2, n, 2).tolist())
        if a != b:
            edges.add((a, b))
    g = P.Graph(n, sorted(edges))
    sol = (rng.random((2, n)) < 0.05).astype(np.uint8)
    sol[1, 1] = 1  # the second hub in S in slot 1
    E = np.array(sorted(edges))

    def worker(comm):
        part = P.partition_rows(n, comm.size)[comm.rank]
        st = P.PartitionedState([g, g], part, solutions=sol)
        out = []
        for b in range(2):
            cand = comm.all_gather(st.cand[b], axis=-1)
            rows, cols = st.local_residual_coo(b)
            out.append((cand, set(zip(rows.tolist(), cols.tolist())), st.local_residual[b]))
        return out
    res = P.run_workers(p, worker)
    for b in range(2):
        alive = E[(sol[b, E[:, 0]] == 0) & (sol[b, E[:, 1]] == 0)]
        want = {(int(u), int(v)) for u, v in alive} | {(int(v), int(u)) for u, v in alive}
        deg = np.bincount(alive.ravel(), minlength=n)
        assert np.array_equal(res[0][b][0], ((deg > 0) & (sol[b] == 0)).astype(np.uint8))
        assert set().union(*(r[b][1] for r in res)) == want
        assert sum(int(r[b][2]) for r in res) == 2 * len(alive)


def test_state_build_coarse_summary_many_nodes():
    """9M nodes: shard_init's shared-memory S summary covers 2^6 nodes per bit
    (the multi-word summary path); candidates and the residual count still
    equal the definition, with a 2,000-entry hub and a 1% solution."""
    rng = np.random.default_rng(11)
    n = 9_000_000
    a = rng.integers(0, n, 60_000)
    b = rng.integers(0, n, 60_000)
    keep = a != b
    pairs = np.unique(np.sort(np.stack([a[keep], b[keep]], 1), axis=1), axis=0)
    hub = np.stack([np.zeros(2000, np.int64), rng.choice(np.arange(1, n), 2000, replace=False)], 1)
    E = np.unique(np.concatenate([pairs, hub]), axis=0)
    g = P.Graph(n, [tuple(e) for e in E.tolist()])
    sol = (rng.random((1, n)) < 0.01).astype(np.uint8)

    def worker(comm):
        st = P.PartitionedState([g], P.partition_rows(n, 1)[0], solutions=sol)
        return st.cand[0].copy(), int(st.local_residual[0])
    cand, resid = P.run_workers(1, worker)[0]
    alive = E[(sol[0, E[:, 0]] == 0) & (sol[0, E[:, 1]] == 0)]
    deg = np.bincount(alive.ravel(), minlength=n)
    assert np.array_equal(cand, ((deg > 0) & (sol[0] == 0)).astype(np.uint8))
    assert resid == 2 * len(alive)


class TestActAndTargets:
    """pkg/tests/test_agent.py:46-112."""

    def test_greedy_zero_params_lowest_index_candidate(self):
        g = P.Graph(4, [(1, 2), (2, 3)])

        def worker(comm):
            env = P.reset(g, comm)
            return P.act(env.state, zero_params(), 0.0, np.random.default_rng(0), comm)
        assert P.run_workers(1, worker) == [1]

    def test_greedy_is_argmax_of_masked_scores_and_p_invariant(self):
        g = P.generate_er(40, 0.2, 13)
        params = P.PolicyParams.initialize(8, 2, seed=21)

        def worker(comm):
            env = P.reset(g, comm)
            a = P.act(env.state, params, 0.0, np.random.default_rng(0), comm)
            emb = P.embed_forward(env.state, params, comm)
            sc = P.masked_scores(P.q_forward(emb, env.state.cand, params, comm), env.state.cand)
            return a, int(np.argmax(comm.all_gather(sc, axis=-1)[0]))
        outs = [P.run_workers(p, worker) for p in (1, 2, 3)]
        ref = outs[0][0][1]
        for res in outs:
            for a, am in res:
                assert a == am == ref

    def test_exploration_uses_the_shared_rng_stream(self):
        g = P.Graph(5, [(0, 1), (1, 2), (2, 3), (3, 4)])

        def worker(comm):
            env = P.reset(g, comm)
            rng = np.random.default_rng(99)
            return [P.act(env.state, zero_params(), 1.0, rng, comm) for _ in range(200)]
        draws = P.run_workers(1, worker)[0]
        rng = np.random.default_rng(99)
        expect = []
        for _ in range(200):
            rng.random()
            expect.append(int(rng.integers(5)))
        assert draws == expect

    def test_targets(self):
        def worker(comm):
            env = P.reset(P.Graph(2, [(0, 1)]), comm)
            env.step(0)
            params = P.PolicyParams.initialize(4, 2, seed=0)
            t_term = P.compute_target(-1.0, env.state, params, comm, 0.9)
            env2 = P.reset(PATH3, comm)
            env2.step(0)
            t0 = P.compute_target(-1.0, env2.state, params, comm, 0.0)
            t = P.compute_target(-1.0, env2.state, params, comm, 0.9)
            emb = P.embed_forward(env2.state, params, comm)
            sc = P.masked_scores(P.q_forward(emb, env2.state.cand, params, comm),
                                 env2.state.cand)
            return t_term, t0, t, float(np.max(sc))
        t_term, t0, t, mx = P.run_workers(1, worker)[0]
        assert t_term == -1.0 and t0 == -1.0
        assert t == -1.0 + 0.9 * mx


class TestReplayAndTraining:
    """pkg/tests/test_agent.py:116-345."""

    def test_snapshot_regenerates_residual(self):
        g = P.Graph(4, [(0, 1), (1, 2), (2, 3)])
        bits = np.array([0, 1, 0, 0], np.uint8)

        def worker(comm):
            t = P.ExperienceTuple(0, P.pack_solution(bits), 2, 0.0)
            st = P.tuples_to_graphs([t], [g], P.partition_rows(4, 1)[0])
            rows, cols = st.local_residual_coo(0)
            return set(zip(rows.tolist(), cols.tolist()))
        assert P.run_workers(1, worker)[0] == {(2, 3), (3, 2)}

    def _setup(self, comm, num_tuples=6, seed=0):
        rng = np.random.default_rng(seed)
        dataset = [P.generate_er(8, 0.4, 100 + i + 10 * seed) for i in range(2)]
        part = P.partition_rows(8, comm.size)[comm.rank]
        buf = P.ReplayBuffer(50)
        for _ in range(num_tuples):
            gi = int(rng.integers(len(dataset)))
            deg = dataset[gi].degrees()
            action = int(rng.choice(np.flatnonzero(deg > 0)))
            buf.add(P.ExperienceTuple(gi, P.pack_solution(np.zeros(8, np.uint8)), action,
                                      float(rng.normal())))
        return dataset, part, buf

    def test_tau_one_is_one_adam_step_and_seeded_runs_match(self):
        def worker(comm):
            dataset, part, buf = self._setup(comm)
            out = []
            for _ in range(2):
                params = P.PolicyParams.initialize(4, 2, seed=1)
                adam = P.AdamState.create(params, lr=1e-3)
                cfg = P.TrainConfig(embed_dim=4, num_layers=2, batch_size=4, tau=1)
                losses = P.train_step(buf, dataset, params, adam, cfg,
                                      np.random.default_rng(42), comm, part)
                out.append((len(losses), adam.step, params))
            return out
        (n1, s1, p1), (n2, s2, p2) = P.run_workers(1, worker)[0]
        assert (n1, s1) == (1, 1)
        for k in PARAM_NAMES:
            assert np.array_equal(getattr(p1, k), getattr(p2, k))

    def test_repeated_iterations_mostly_decrease_loss(self):
        def worker(comm):
            down = total = 0
            for seed in range(10):
                dataset, part, buf = self._setup(comm, seed=seed)
                params = P.PolicyParams.initialize(4, 2, seed=seed, scale=0.3)
                adam = P.AdamState.create(params, lr=1e-3)
                cfg = P.TrainConfig(embed_dim=4, num_layers=2, batch_size=6, tau=4, seed=seed)
                losses = P.train_step(buf, dataset, params, adam, cfg,
                                      np.random.default_rng(seed), comm, part)
                down += sum(b <= a for a, b in zip(losses, losses[1:]))
                total += len(losses) - 1
            return down / total
        assert P.run_workers(1, worker)[0] >= 0.75

    def test_train_loop_ranks_stay_synchronized(self):
        dataset = [P.generate_er(8, 0.35, 300 + i) for i in range(2)]

        def worker(comm):
            cfg = P.TrainConfig(embed_dim=4, num_layers=2, batch_size=4, tau=1, seed=7,
                                eps_decay_steps=10)
            params, _ = P.train(dataset, cfg, comm, max_steps=12)
            return params
        outs = P.run_workers(2, worker)
        for k in PARAM_NAMES:
            assert np.array_equal(getattr(outs[0], k), getattr(outs[1], k))


class TestGradients:
    """pkg/tests/test_policy.py:196-262: fp64 central differences."""

    def _case(self, rng, n, k, layers, batch):
        graphs, sols, actions = [], [], []
        for _ in range(batch):
            while True:
                g = P.generate_er(n, 0.45, int(rng.integers(1 << 30)))
                if g.num_edges == 0:
                    continue
                deg = g.degrees()
                sol = np.where((rng.random(n) < 0.3) & (deg > 0), 1, 0).astype(np.uint8)
                st_ok = [v for v in range(n) if not sol[v] and any(
                    (u == v and not sol[w]) or (w == v and not sol[u]) for u, w in g.edge_array)]
                if st_ok:
                    break
            graphs.append(g)
            sols.append(sol)
            actions.append(int(rng.choice(st_ok)))
        return graphs, np.stack(sols), np.array(actions), rng.normal(size=batch)

    def test_matches_finite_differences(self):
        rng = np.random.default_rng(2024)

        def worker(comm):
            worst_all = 0.0
            for _ in range(4):
                n, k = int(rng.integers(4, 9)), int(rng.choice([2, 4]))
                layers, batch = int(rng.choice([1, 2])), int(rng.choice([1, 3]))
                graphs, sols, actions, targets = self._case(rng, n, k, layers, batch)
                shapes = param_shapes(k)
                arrays = {nm: rng.uniform(0.3, 0.9, shapes[nm]) * rng.choice([-1.0, 1.0], shapes[nm])
                          for nm in PARAM_NAMES}
                params = P.PolicyParams(num_layers=layers, **arrays)
                st = P.PartitionedState(graphs, P.partition_rows(n, 1)[0], solutions=sols,
                                        dtype=np.float64)

                def loss_fn():
                    return P.loss_and_gradients(st, actions, targets, params, comm)[0]
                _, analytic = P.loss_and_gradients(st, actions, targets, params, comm)
                h = 1e-3
                for nm in PARAM_NAMES:
                    flat = getattr(params, nm).ravel()
                    fd = np.zeros_like(flat)
                    for i in range(flat.size):
                        orig = flat[i]
                        flat[i] = orig + h
                        up = loss_fn()
                        flat[i] = orig - h
                        down = loss_fn()
                        flat[i] = orig
                        fd[i] = (up - down) / (2 * h)
                    worst = relative_error(analytic[nm].ravel(), fd, floor=1e-5).max()
                    worst_all = max(worst_all, worst)
            return worst_all
        assert P.run_workers(1, worker)[0] < 1e-4

    def test_zero_loss_zero_grads(self):
        rng = np.random.default_rng(5)

        def worker(comm):
            graphs, sols, actions, _ = self._case(rng, 6, 4, 2, 2)
            params = P.PolicyParams.initialize(4, 2, seed=3, dtype=np.float64)
            st = P.PartitionedState(graphs, P.partition_rows(6, 1)[0], solutions=sols,
                                    dtype=np.float64)
            emb = P.embed_forward(st, params, comm)
            onehot = np.zeros((2, 6), np.uint8)
            onehot[np.arange(2), actions] = 1
            sc = P.q_forward(emb, onehot, params, comm)
            targets = np.array([sc[i, a] for i, a in enumerate(actions)])
            return P.loss_and_gradients(st, actions, targets, params, comm)
        loss, grads = P.run_workers(1, worker)[0]
        assert loss == 0.0 and all(not grads[n].any() for n in PARAM_NAMES)
