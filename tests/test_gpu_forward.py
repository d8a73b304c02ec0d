"""GPU parity of the forward path against the C++ op-order oracle (bitwise)."""
import numpy as np
import pytest

import paper_2105_08764_b200 as P
from oracle import cref

pytestmark = pytest.mark.gpu


def _forward_gpu(g, params, sol=None):
    def worker(comm):
        part = P.partition_rows(g.num_nodes, comm.size)[comm.rank]
        st = P.PartitionedState([g], part, solutions=None if sol is None else sol[None],
                                dtype=params.dtype)
        emb = P.embed_forward(st, params, comm)
        h = np.asarray(emb)[0].T.copy()
        sc = P.q_forward(emb, st.cand, params, comm)[0]
        return h, sc, st.cand[0].copy()
    return P.run_workers(1, worker)[0]


@pytest.mark.parametrize("n,m,K,L,seed,solfrac,dtype", [
    (1000, 4, 64, 5, 0, 0.0, np.float32),
    (1000, 4, 64, 5, 0, 0.1, np.float32),
    (800, 4, 32, 2, 1, 0.05, np.float32),
    (300, 3, 8, 3, 2, 0.1, np.float32),
    (500, 5, 16, 4, 3, 0.1, np.float64),
    (3000, 8, 64, 5, 4, 0.2, np.float32),
])
def test_forward_bitwise_vs_oracle(n, m, K, L, seed, solfrac, dtype):
    g = P.generate_ba(n, m, seed)
    params = P.PolicyParams.initialize(K, L, seed=seed, dtype=dtype)
    rng = np.random.default_rng(seed)
    sol = (rng.random(n) < solfrac).astype(np.uint8)
    h_gpu, s_gpu, cand_gpu = _forward_gpu(g, params, sol)
    rp, cols = g.csr_arrays()
    h, gsum, u1, cand, sc = cref.forward(rp, cols, sol, params.as_dict(), L, dtype=dtype)
    assert np.array_equal(cand_gpu, cand)
    assert np.array_equal(h_gpu, h), np.abs(h_gpu - h).max()
    assert np.array_equal(s_gpu, sc), np.abs(s_gpu - sc).max()


def _hub_graph():
    """BA(3000,4) plus a star: node 7 joined to 5000 others, so node 7 (and
    nothing else) exceeds the hub degree and takes the cooperative kernel."""
    base = P.generate_ba(6000, 4, 5)
    extra = np.stack([np.full(5000, 7), np.arange(1000, 6000)], axis=1)
    return P.Graph(6000, np.concatenate([base.edge_array, extra]))


@pytest.mark.parametrize("make", ["hub", "rmat16"])
def test_hub_rows_bitwise_vs_oracle(make):
    g = _hub_graph() if make == "hub" else P.generate_rmat(16, 16, 0)
    rp, cols = g.csr_arrays()
    assert np.diff(rp).max() > 4096
    params = P.PolicyParams.initialize(64, 5, seed=1)
    sol = (np.random.default_rng(2).random(g.num_nodes) < 0.05).astype(np.uint8)
    h_gpu, s_gpu, cand_gpu = _forward_gpu(g, params, sol)
    h, _, _, cand, sc = cref.forward(rp, cols, sol, params.as_dict(), 5)
    assert np.array_equal(cand_gpu, cand)
    assert np.array_equal(h_gpu, h)
    assert np.array_equal(s_gpu, sc)


@pytest.mark.parametrize("make", ["ba", "hub"])
def test_degree_table_round2_equals_plain_round(make, monkeypatch):
    """Round 2 from the per-degree table of round-1 outputs
    (s2v_embed_round2_table) gives the bits of the plain round reading h1,
    for a batch of slots with partial solutions, with and without hub rows."""
    gs = [_hub_graph(), P.generate_ba(6000, 4, 9)] if make == "hub" else \
        [P.generate_ba(4000, 6, 1), P.generate_ba(4000, 3, 2), P.generate_ba(4000, 8, 3)]
    n = gs[0].num_nodes
    params = P.PolicyParams.initialize(64, 5, seed=3)
    rng = np.random.default_rng(4)
    sol = (rng.random((len(gs), n)) < 0.1).astype(np.uint8)

    def run():
        def worker(comm):
            part = P.partition_rows(n, 1)[0]
            st = P.PartitionedState(gs, part, solutions=sol)
            emb = P.embed_forward(st, params, comm)
            return np.asarray(emb).copy(), P.q_forward(emb, st.cand, params, comm)
        return P.run_workers(1, worker)[0]

    monkeypatch.setenv("S2V_DEG_TABLE", "1")
    h_t, s_t = run()
    monkeypatch.setenv("S2V_DEG_TABLE", "0")
    h_p, s_p = run()
    assert np.array_equal(h_t, h_p)
    assert np.array_equal(s_t, s_p)
    rp, cols = gs[1].csr_arrays()
    h_o = cref.forward(rp, cols, sol[1], params.as_dict(), 5)[0]
    assert np.array_equal(h_t[1].T, h_o)  # (scores at B > 1 follow the batched u1 order)


def test_big_table_edge_degree_pass_bitwise(monkeypatch):
    """A degree table above 8 MB (a 40,000-leaf star: max degree > 32K)
    takes the streaming edge-degree pass before round 2; embeddings and
    scores stay bitwise equal to the oracle and to the in-gather lookup."""
    base = P.generate_ba(50000, 4, 8)
    star = np.stack([np.full(40000, 3), np.arange(10000, 50000)], axis=1)
    g = P.Graph(50000, np.concatenate([base.edge_array, star]))
    rp, cols = g.csr_arrays()
    assert (int(np.diff(rp).max()) + 2) * 256 > 8 << 20
    params = P.PolicyParams.initialize(64, 5, seed=4)
    sol = (np.random.default_rng(5).random(g.num_nodes) < 0.02).astype(np.uint8)
    monkeypatch.setenv("S2V_EDGE_DEG", "1")
    h_gpu, s_gpu, cand_gpu = _forward_gpu(g, params, sol)
    h, _, _, cand, sc = cref.forward(rp, cols, sol, params.as_dict(), 5)
    assert np.array_equal(cand_gpu, cand)
    assert np.array_equal(h_gpu, h)
    assert np.array_equal(s_gpu, sc)
