"""Restatements of the reference tests that tests/ref_suite does not run
verbatim (tests/ref_suite/conftest.py ADAPTED), adapted to the halo design.

pkg/tests/test_policy.py:290-313 pins the reference's comm pattern: per
embedding round an all-reduce of the B*K*N partial neighbour sums.  Here each
round all-gathers the N_loc*K rows every rank owns (rows_max per rank, the
in-place halo chunk), so the per-call element count is B*rows_max*K; the
call counts (2L embed_fwd, 2 q_fwd, 1 grad) and the fp64 gradient pack size
are unchanged, and the backward adds its dg (q_bwd) and L-1 dm (embed_bwd)
exchanges."""
import numpy as np
import pytest

import paper_2105_08764_b200 as P

pytestmark = pytest.mark.gpu


def test_embed_q_and_grad_call_counts_halo_design():
    g = P.generate_er(10, 0.3, 1)
    params = P.PolicyParams.initialize(4, 3, seed=0)
    group = P.WorkerGroup(2)

    def worker(comm):
        part = P.partition_rows(g.num_nodes, comm.size)[comm.rank]
        state = P.PartitionedState([g], part, dtype=np.float32)
        embed = P.embed_forward(state, params, comm)
        P.q_forward(embed, state.cand, params, comm)
        P.loss_and_gradients(state, np.array([0]), np.array([0.0]), params, comm)
        return state.rows_max
    rows_max = P.run_workers(2, worker, group=group)[0]
    stats = group.stats_snapshot()
    k, L = params.embed_dim, params.num_layers
    assert stats["embed_fwd"].calls == 2 * L
    assert stats["q_fwd"].calls == 2
    assert stats["grad"].calls == 1
    assert rows_max == 5
    assert stats["embed_fwd"].elements // stats["embed_fwd"].calls == 1 * rows_max * k
    assert stats["q_fwd"].elements // stats["q_fwd"].calls == 1 * k
    assert stats["grad"].elements == 4 * k * k + 4 * k + 1
    assert stats["q_bwd"].calls == 1 and stats["q_bwd"].elements == k
    assert stats["embed_bwd"].calls == L - 1
    assert stats["embed_bwd"].elements == (L - 1) * rows_max * k
