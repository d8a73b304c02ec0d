"""CPU: the oracle is pinned against golden vectors produced by the reference
itself (oracle/make_golden.py, tests/golden/) and the reference's own dyadic
known-answer vectors (pkg/tests/test_policy.py:16-42)."""
import json
from pathlib import Path

import numpy as np
import pytest

import paper_2105_08764_b200 as P
from oracle import cref, port

GOLD = Path(__file__).resolve().parent / "golden"
FWD = ["fwd_ba1000_k64_l5", "fwd_ba1000_k64_l5_sol10", "fwd_ba800_k32_l2", "fwd_ba5000_m8_k64_l5"]


@pytest.mark.parametrize("name", FWD)
def test_cpp_oracle_forward_bitwise_vs_reference(name):
    z = np.load(GOLD / f"{name}.npz")
    g = P.generate_ba(int(z["n"]), int(z["m"]), int(z["seed"]))
    params = P.PolicyParams.initialize(int(z["K"]), int(z["L"]), seed=int(z["pseed"]))
    rp, cols = g.csr_arrays()
    h, gs, u1, cand, sc = cref.forward(rp, cols, z["sol"], params.as_dict(), int(z["L"]))
    assert np.array_equal(h, z["h"])
    assert np.array_equal(gs, z["g"])
    assert np.array_equal(u1, z["u1"])
    assert np.array_equal(cand, z["cand"])
    assert np.array_equal(sc, z["scores"])


@pytest.mark.parametrize("name", FWD[:3])
def test_port_forward_bitwise_vs_reference(name):
    z = np.load(GOLD / f"{name}.npz")
    g = P.generate_ba(int(z["n"]), int(z["m"]), int(z["seed"]))
    params = P.PolicyParams.initialize(int(z["K"]), int(z["L"]), seed=int(z["pseed"]))
    st = port.ResidualState([g.edge_array], g.num_nodes, solutions=z["sol"][None])
    h = port.embed(st, params.as_dict(), int(z["L"]))
    s = port.scores(h, st.cand, params.as_dict())
    assert np.array_equal(h[0].T, z["h"])
    assert np.array_equal(s[0], z["scores"])


SOLVES = {
    "solve_ba1000_k64_l5": (lambda: [P.generate_ba(1000, 4, 0)], None),
    "solve_ba1000_k64_l5_single": (lambda: [P.generate_ba(1000, 4, 0)],
                                   {"thresholds": (), "fallback": 1}),
    "solve_batch3_k32_l2": (lambda: [P.generate_ba(800, 4, s) for s in (1, 2, 3)], None),
    "solve_er300_fixed8_k16_l3": (lambda: [P.generate_er(300, 0.05, 7)],
                                  {"thresholds": (), "fallback": 8}),
}


@pytest.mark.parametrize("name", list(SOLVES))
def test_port_solve_matches_reference_trajectory(name):
    z = np.load(GOLD / f"{name}.npz")
    make, sched = SOLVES[name]
    graphs = make()
    params = P.PolicyParams.initialize(int(z["K"]), int(z["L"]), seed=int(z["pseed"]))
    res = port.solve([g.edge_array for g in graphs], graphs[0].num_nodes, params.as_dict(),
                     int(z["L"]), sched)
    offs = np.concatenate([[0], np.cumsum(z["cover_lens"])])
    for b, (cover, evals, skipped, trace) in enumerate(res):
        assert cover == z["covers"][offs[b]:offs[b + 1]].tolist()
        assert evals == int(z["evals"][b]) and skipped == int(z["skipped"][b])
    if len(res) == 1:
        flat = [v for picks in res[0][3] for v in picks]
        assert flat == z["pick_flat"].tolist()


@pytest.mark.parametrize("name", ["train_ba1000_b4_k64_l5", "train_ba600_b3_k16_l3_f64"])
def test_port_training_step_bitwise_vs_reference(name):
    z = np.load(GOLD / f"{name}.npz")
    n, m, B, L, tau = (int(z[k]) for k in ("n", "m", "B", "L", "tau"))
    graphs = [P.generate_ba(n, m, 100 + i) for i in range(B)]
    theta = {k: z[f"p0_{k}"].copy() for k in port.NAMES}
    edges = [g.edge_array for g in graphs]
    t = port.batch_targets(edges, n, z["snaps"], z["actions"], theta, L, 0.9).astype(
        theta["theta1"].dtype)
    assert np.array_equal(t, z["targets"])
    st = port.ResidualState(edges, n, solutions=z["snaps"], dtype=theta["theta1"].dtype)
    mom = {k: np.zeros_like(v) for k, v in theta.items()}
    vel = {k: np.zeros_like(v) for k, v in theta.items()}
    step, losses = 0, []
    for it in range(tau):
        loss, grads = port.loss_and_grads(st, z["actions"], t, theta, L)
        if it == 0:
            for k in port.NAMES:
                assert np.array_equal(grads[k], z[f"g0_{k}"]), k
        step = port.adam(theta, grads, mom, vel, step, 1e-5)
        losses.append(loss)
    assert np.array_equal(np.array(losses), z["losses"])
    for k in port.NAMES:
        assert np.array_equal(theta[k], z[f"p1_{k}"]), k


def _hand_params(kat, layers):
    return {k: np.asarray(v, dtype=np.float64) for k, v in kat["HAND_THETA"].items()}, layers


def test_cpp_oracle_dyadic_kats():
    kat = json.loads((GOLD / "kat_dyadic.json").read_text())
    theta = {k: np.asarray(v, dtype=np.float64) for k, v in kat["HAND_THETA"].items()}
    path = P.Graph(3, [(0, 1), (1, 2)])
    rp, cols = path.csr_arrays()
    sol = np.zeros(3, np.uint8)
    assert np.array_equal(cref.embed(rp, cols, sol, theta, 1, np.float64).T,
                          kat["EXPECTED_PATH_L1"])
    h2 = cref.embed(rp, cols, sol, theta, 2, np.float64)
    assert np.array_equal(h2.T, kat["EXPECTED_PATH_L2"])
    u1 = (cref.colsum(h2)[None] @ theta["theta5"].T)[0]
    assert np.array_equal(cref.scores(h2, np.ones(3, np.uint8), theta, u1),
                          kat["EXPECTED_PATH_SCORES"])
    assert np.array_equal(cref.scores(h2, np.array([1, 0, 1], np.uint8), theta, u1),
                          kat["EXPECTED_PATH_SCORES_EXTRACT"])
    cyc = P.Graph(5, [(0, 1), (1, 2), (2, 3), (3, 4), (0, 4)])
    rp, cols = cyc.csr_arrays()
    sol = np.array([1, 0, 0, 0, 0], np.uint8)
    h = cref.embed(rp, cols, sol, theta, 2, np.float64)
    assert np.array_equal(h.T, kat["EXPECTED_CYCLE_L2"])


def test_native_ba_generator_is_the_reference_graph():
    # edge count formula of graphs.py:125-157 and the golden forward (which
    # used the reference's own generate_ba) pin the generator
    for n, d in ((1000, 4), (5000, 8), (300, 1)):
        g = P.generate_ba(n, d, 3)
        assert g.num_edges == d * (d - 1) // 2 + d * (n - d)
        rp, cols = g.csr_arrays()
        assert np.all(np.diff(rp) >= 1)
        for v in (0, n // 2, n - 1):
            row = cols[rp[v]:rp[v + 1]]
            assert np.all(np.diff(row) > 0)


def _edge_sha(g):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(g.edge_array, dtype=np.int64).tobytes()).hexdigest()


@pytest.mark.parametrize("case", range(3))
def test_native_ba_generator_equals_reference_bytes(case):
    """Native generate_ba (csrc/s2v_graphgen.cu) == the reference's
    generate_ba (pkg/src/graphrl/graphs.py:125-157), edge array byte for
    byte, up to BA(100000,16): fixtures/generators.json was written by the
    reference itself (oracle/make_golden.py gen)."""
    gold = json.loads((GOLD / "generators.json").read_text())["ba"][case]
    g = P.generate_ba(gold["n"], gold["d"], gold["seed"])
    assert g.num_edges == gold["edges"]
    assert _edge_sha(g) == gold["sha256"]


@pytest.mark.parametrize("case", range(2))
def test_er_generator_equals_reference_bytes(case):
    gold = json.loads((GOLD / "generators.json").read_text())["er"][case]
    g = P.generate_er(gold["n"], gold["rho"], gold["seed"])
    assert g.num_edges == gold["edges"]
    assert _edge_sha(g) == gold["sha256"]


@pytest.mark.parametrize("scale,chunk", [(10, 1 << 23), (14, 1 << 23), (14, 1 << 12)])
def test_native_rmat_equals_numpy_definition(scale, chunk):
    """Native R-MAT (PCG64 jump-ahead across threads) == generate_rmat_numpy,
    the numpy statement of the definition, including multi-chunk draws."""
    a = P.generate_rmat(scale, 16, 0, chunk=chunk)
    b = P.graphs.generate_rmat_numpy(scale, 16, 0, chunk=chunk)
    assert a.num_nodes == b.num_nodes
    assert np.array_equal(a.edge_array, b.edge_array)


@pytest.mark.parametrize("case", range(3))
def test_oracle_ba_generator_equals_reference_bytes(case):
    """The C restatement that builds the reference arm's input graph
    (oracle/ba_oracle.c) == the reference's generate_ba, byte for byte."""
    import hashlib
    gold = json.loads((GOLD / "generators.json").read_text())["ba"][case]
    e = cref.generate_ba_edges(gold["n"], gold["d"], gold["seed"])
    assert e.shape[0] == gold["edges"]
    assert hashlib.sha256(np.ascontiguousarray(e).tobytes()).hexdigest() == gold["sha256"]
