"""Node-sharded (P > 1) execution on the GPU: P thread-ranks (sharing the one
B200 of the test box, or one GPU each) run the row-partitioned shards with the
in-process device transport.  The halo design makes every result bitwise
P-invariant and equal to the P = 1 oracle -- stronger than the reference,
whose rank-ordered partial sums differ across P."""
from pathlib import Path

import numpy as np
import pytest

import paper_2105_08764_b200 as P
from oracle import cref, port
from reference_math import scale_error

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("p", [2, 3, 4])
def test_forward_bitwise_at_any_p(p):
    g = P.generate_ba(1000, 4, 0)
    params = P.PolicyParams.initialize(64, 5, seed=0)
    sol = (np.random.default_rng(3).random(1000) < 0.1).astype(np.uint8)

    def worker(comm):
        part = P.partition_rows(1000, comm.size)[comm.rank]
        st = P.PartitionedState([g], part, solutions=sol[None])
        emb = P.embed_forward(st, params, comm)
        sc = P.q_forward(emb, st.cand, params, comm)
        return comm.all_gather(emb, axis=-1), comm.all_gather(sc, axis=-1)
    outs = P.run_workers(p, worker)
    rp, cols = g.csr_arrays()
    h, _, _, _, sc = cref.forward(rp, cols, sol, params.as_dict(), 5)
    for emb, scores in outs:
        assert np.array_equal(emb[0].T, h)
        assert np.array_equal(scores[0], sc)


@pytest.mark.parametrize("p", [2, 4])
def test_solve_trajectory_is_the_p1_reference_at_any_p(p):
    gold = np.load(GOLD / "solve_ba1000_k64_l5.npz")
    g = P.generate_ba(1000, 4, 0)
    params = P.PolicyParams.initialize(64, 5, seed=0)
    res = P.run_workers(p, lambda comm: P.solve([g], params, comm))
    for (r,) in res:
        assert r.cover == gold["covers"].tolist()
        assert r.policy_evals == int(gold["evals"][0])
        assert r.skipped == int(gold["skipped"][0])


def test_batched_solve_p3():
    gold = np.load(GOLD / "solve_batch3_k32_l2.npz")
    graphs = [P.generate_ba(800, 4, s) for s in (1, 2, 3)]
    params = P.PolicyParams.initialize(32, 2, seed=1)
    res = P.run_workers(3, lambda comm: P.solve(graphs, params, comm))[0]
    offs = np.concatenate([[0], np.cumsum(gold["cover_lens"])])
    for b, r in enumerate(res):
        assert r.cover == gold["covers"][offs[b]:offs[b + 1]].tolist()


@pytest.mark.parametrize("p", [2, 3])
def test_gradients_p_invariant_and_replicas_identical(p):
    rng = np.random.default_rng(7)
    n, B, K, L = 300, 3, 16, 3
    graphs = [P.generate_ba(n, 3, 70 + i) for i in range(B)]
    sols = (rng.random((B, n)) < 0.15).astype(np.uint8)
    ps = port.ResidualState([g.edge_array for g in graphs], n, solutions=sols)
    actions = np.array([int(np.flatnonzero(ps.cand[b])[0]) for b in range(B)])
    targets = rng.normal(size=B).astype(np.float32)
    params = P.PolicyParams.initialize(K, L, seed=2, orientation="symmetric")

    def worker(comm):
        part = P.partition_rows(n, comm.size)[comm.rank]
        st = P.PartitionedState(graphs, part, solutions=sols)
        return P.loss_and_gradients(st, actions, targets, params, comm)
    base_loss, base = P.run_workers(1, worker)[0]
    outs = P.run_workers(p, worker)
    for loss, grads in outs:
        assert abs(loss - base_loss) <= 1e-6 * max(1.0, abs(base_loss))
        for k in P.PARAM_NAMES:
            assert scale_error(grads[k], base[k]).max() < 1e-5, k
    for loss, grads in outs[1:]:
        assert loss == outs[0][0]
        for k in P.PARAM_NAMES:
            assert np.array_equal(grads[k], outs[0][1][k])


def test_owner_side_rejection_under_p2():
    g = P.Graph(4, [(0, 1), (1, 2), (2, 3)])

    def worker(comm):
        part = P.partition_rows(4, comm.size)[comm.rank]
        st = P.PartitionedState([g], part)
        st.apply_action(1)
        st.apply_action(1)
    with pytest.raises(P.InvalidActionError, match="already in the solution"):
        P.run_workers(2, worker)


@pytest.mark.parametrize("kind,dtype", [(2, np.float32), (1, np.float64), (0, np.int64)])
def test_device_allreduce_is_rank_ordered(kind, dtype):
    """The peer transport's all-reduce sums rank 0, then += rank 1, rank 2 on
    the device (collective.py:114-116): values chosen so that fp addition
    order shows, and every rank holds the same bits as the host Comm's sum."""
    import torch
    from paper_2105_08764_b200.device import stream_ptr
    rng = np.random.default_rng(11)
    vals = [(rng.standard_normal(1000) * 10.0 ** rng.integers(-6, 7, 1000)).astype(dtype)
            if kind else rng.integers(-2**40, 2**40, 1000) for _ in range(3)]
    want = vals[0].copy()
    for v in vals[1:]:
        want += v

    def worker(comm):
        dc = comm.device_comm()
        assert dc.supports_push
        t = torch.from_numpy(vals[comm.rank].copy()).cuda()
        for _ in range(3):  # alternating scratch buffers, repeated use
            u = t.clone()
            dc.allreduce(u.data_ptr(), u.numel(), kind, stream_ptr())
        host = comm.all_reduce_sum(vals[comm.rank])
        return u.cpu().numpy(), host
    for dev_sum, host_sum in P.run_workers(3, worker):
        assert np.array_equal(dev_sum, want)
        assert np.array_equal(dev_sum, host_sum)


@pytest.mark.parametrize("p", [2, 3])
def test_device_tau_loop_at_p_ranks(p):
    """train_iterations (the device tau loop) at P thread-ranks: dg and the
    gradient pack are all-reduced on the device, replicas end bit-identical
    and equal to P = 1 within the gradient bar."""
    rng = np.random.default_rng(5)
    n, B, K, L, tau = 400, 2, 32, 3, 3
    graphs = [P.generate_ba(n, 4, 90 + i) for i in range(B)]
    sols = (rng.random((B, n)) < 0.1).astype(np.uint8)
    ps = port.ResidualState([g.edge_array for g in graphs], n, solutions=sols)
    actions = np.array([int(np.flatnonzero(ps.cand[b])[1]) for b in range(B)])
    targets = rng.normal(size=B).astype(np.float32)

    def worker(comm):
        params = P.PolicyParams.initialize(K, L, seed=4)
        adam = P.AdamState.create(params, lr=1e-3)
        part = P.partition_rows(n, comm.size)[comm.rank]
        st = P.PartitionedState(graphs, part, solutions=sols)
        losses = P.policy.train_iterations(st, actions, targets, params, adam, tau, comm)
        return losses, params
    (l1, p1), = P.run_workers(1, worker)
    outs = P.run_workers(p, worker)
    for losses, params in outs:
        assert np.allclose(losses, l1, rtol=1e-5)
        for k in P.PARAM_NAMES:
            assert scale_error(getattr(params, k), getattr(p1, k)).max() < 1e-4, k
    for losses, params in outs[1:]:
        assert losses == outs[0][0]
        for k in P.PARAM_NAMES:
            assert np.array_equal(getattr(params, k), getattr(outs[0][1], k))


@pytest.mark.parametrize("p", [2, 3])
def test_compacted_episode_at_p_ranks(p, monkeypatch):
    """Residual-row compaction at P > 1 (every rank visits only its rows with
    rdeg > 0; the gathered global sum takes dead rows from the h1 table,
    classified by every rank's e12 rows; each rank's compact CSR tests S of
    every rank's rows, kept by s2v_sol_mark): the whole episode's pick/apply
    trace equals the P = 1 loop over every row.  R-MAT with isolated nodes."""
    from paper_2105_08764_b200.inference import DeviceEpisode
    monkeypatch.setattr(DeviceEpisode, "COMPACT_MIN_ROWS", 0)
    g = P.generate_rmat(13, 16, 2)
    params = P.PolicyParams.initialize(64, 5, seed=6)
    sched = P.SelectionSchedule.adaptive()

    def run(compact):
        def worker(comm):
            st = P.PartitionedState([g], P.partition_rows(g.num_nodes, comm.size)[comm.rank])
            ep = DeviceEpisode(st, params, comm, sched, 4, use_graph=False, compact=compact)
            assert ep.compact == compact
            trace = []
            while True:
                tp, ta, te, active = ep.run_chunk()
                trace.append((tp.copy(), ta.copy(), te.copy()))
                if not active.any():
                    break
            return trace, ep.active_count(), getattr(ep, "csr_builds", 0)
        return P.run_workers(comm_size[0], worker)

    comm_size = [1]
    (t_f, _, _), = run(False)
    comm_size[0] = p
    outs = run(True)
    for trace, n_act, csr_builds in outs:
        assert csr_builds > 0  # the compact CSR was read at P > 1
        assert len(trace) == len(t_f)
        for (a, b, c), (x, y, z) in zip(trace, t_f):
            assert np.array_equal(a, x) and np.array_equal(b, y) and np.array_equal(c, z)
        assert n_act < g.num_nodes // p + 1  # the list did shrink


@pytest.mark.parametrize("p", [2, 3])
def test_d1_schedule_is_stepwise_argmax_at_p_ranks(p):
    """The reference's equivalence (pkg/tests/test_inference.py:84-110) at
    P ranks: the d = 1 schedule through solve() (the device episode loop,
    keys merged across ranks) picks exactly the stepwise argmax of the
    all-gathered masked scores (env.step through the public API), on a
    BA graph large enough that every rank owns hubs and leaves."""
    g = P.generate_ba(600, 3, 21)
    params = P.PolicyParams.initialize(16, 3, seed=3)

    def manual(comm):
        env = P.reset(g, comm)
        picks = []
        while not env.terminated:
            emb = P.embed_forward(env.state, params, comm)
            sc = P.q_forward(emb, env.state.cand, params, comm)
            gl = comm.all_gather(P.masked_scores(sc, env.state.cand), axis=-1)[0]
            v = int(np.argmax(gl))
            env.step(v)
            picks.append(v)
        return picks

    def via_solve(comm):
        (res,) = P.solve([g], params, comm, schedule=P.SelectionSchedule.single())
        return res
    picks = P.run_workers(p, manual)
    res = P.run_workers(p, via_solve)
    for pk, r in zip(picks, res):
        assert pk == picks[0]
        assert r.cover == sorted(pk)
        assert r.policy_evals == len(pk)


@pytest.mark.parametrize("p,inc_cap", [(2, 0.25), (3, 0.25), (2, 0.0)])
def test_incremental_episode_at_p_ranks(p, inc_cap, monkeypatch):
    """The incremental forward at P > 1 (frontier levels built from
    all-gathered bitmaps, every rank recomputing only its frontier rows, the
    global sum refreshing only leaves of changed nodes), switched on from
    the first compaction: the whole episode's trace equals the P = 1 loop
    over every row; inc_cap = 0 makes every local frontier overflow."""
    from paper_2105_08764_b200.inference import DeviceEpisode
    monkeypatch.setattr(DeviceEpisode, "COMPACT_MIN_ROWS", 0)
    g = P.generate_rmat(13, 16, 4)
    params = P.PolicyParams.initialize(64, 5, seed=8)
    sched = P.SelectionSchedule.adaptive()

    def run(world, compact):
        def worker(comm):
            st = P.PartitionedState([g], P.partition_rows(g.num_nodes, comm.size)[comm.rank])
            ep = DeviceEpisode(st, params, comm, sched, 4, use_graph=False, compact=compact)
            trace = []
            while True:
                tp, ta, te, active = ep.run_chunk()
                trace.append((tp.copy(), ta.copy(), te.copy()))
                if not active.any():
                    break
            return trace, (ep._mode[2] if compact else None)
        return P.run_workers(world, worker)

    (t_f, _), = run(1, False)
    monkeypatch.setattr(DeviceEpisode, "INC_RATIO", 1e9)
    monkeypatch.setattr(DeviceEpisode, "INC_SLOWER", float("inf"))  # no timing fallback
    monkeypatch.setattr(DeviceEpisode, "LIST_FRAC", 1.0)
    monkeypatch.setattr(DeviceEpisode, "INC_CAP", inc_cap)
    if inc_cap == 0.0:
        monkeypatch.setattr(DeviceEpisode, "INC_MIN", 0)
    for trace, inc_used in run(p, True):
        assert inc_used
        assert len(trace) == len(t_f)
        for i, ((a, b, c), (x, y, z)) in enumerate(zip(trace, t_f)):
            assert np.array_equal(a, x) and np.array_equal(b, y) and np.array_equal(c, z), i


@pytest.mark.parametrize("p", [2, 3])
def test_device_solve_step_at_p_ranks(p, monkeypatch):
    """solve_step at P > 1 merges every rank's top-d keys and sums the apply
    info on the device (_solve_step_device): picks, applied flags, the
    solution bits and the residual counts equal the P = 1 device path and
    the host-merge path at P ranks, step for step (adaptive d, B = 32 --
    a device-u1 shape -- with inactive slots)."""
    from paper_2105_08764_b200 import inference as inf
    graphs = [P.generate_ba(500, 4, 40 + i) for i in range(32)]
    params = P.PolicyParams.initialize(32, 3, seed=2)
    sched = P.SelectionSchedule.adaptive()
    active = np.ones(32, bool)
    active[[1, 30]] = False

    def run(world, device):
        def worker(comm):
            if not device:
                monkeypatch.setattr(inf, "_device_loop_ok", lambda *a: False)
            else:
                assert inf._device_loop_ok(P.PartitionedState(
                    graphs, P.partition_rows(500, comm.size)[comm.rank]), params, comm, sched)
            st = P.PartitionedState(graphs, P.partition_rows(500, comm.size)[comm.rank])
            out = [inf.solve_step(st, params, comm, sched, active) for _ in range(4)]
            sol = comm.all_gather(st.sol.copy(), axis=-1)
            return out, sol, st.residual_counts(comm)
        try:
            return P.run_workers(world, worker)
        finally:
            monkeypatch.undo()
    ref_out, ref_sol, ref_res = run(1, True)[0]
    for device in (True, False):
        for out, sol, res in run(p, device):
            for (pd, ad), (pr, ar) in zip(out, ref_out):
                assert np.array_equal(pd, pr) and np.array_equal(ad, ar)
            assert np.array_equal(sol, ref_sol) and np.array_equal(res, ref_res)
