"""Device build of the shard structure (s2v_shard_structure) against the
numpy restatement of state.py:89-105 / 115-122 it replaced: every array bit
for bit, at P = 1, 2, 3, on a BA graph and on an R-MAT graph with isolated
nodes and hub rows."""
import numpy as np
import pytest

import paper_2105_08764_b200 as P
from paper_2105_08764_b200 import state as S

pytestmark = pytest.mark.gpu


def numpy_structure(graph, part):
    n, p = graph.num_nodes, part.num_workers
    row_ptr_g, cols_g = graph.csr_arrays()
    lo, hi = int(row_ptr_g[part.row_start]), int(row_ptr_g[part.row_stop])
    row_ptr = row_ptr_g[part.row_start:part.row_stop + 1] - lo
    nbr = cols_g[lo:hi]
    cols0 = (S.phys_rows(n, p)[nbr] if p > 1 else nbr).astype(np.int32)
    local_row = np.repeat(np.arange(part.num_rows, dtype=np.int32), np.diff(row_ptr))
    order = np.argsort(nbr, kind="stable")
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(nbr, minlength=n), out=col_ptr[1:])
    deg = np.diff(row_ptr)
    return dict(row_ptr=row_ptr, cols0=cols0, col_ptr=col_ptr, col_ent=order.astype(np.int64),
                col_row=local_row[order], order=np.argsort(-deg, kind="stable").astype(np.int32),
                n_hub=int(np.count_nonzero(deg > P._lib.HUB_DEGREE)),
                max_deg=int(deg.max()) if len(deg) else 0)


@pytest.mark.parametrize("gen", ["ba", "rmat"])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_device_structure_equals_numpy(gen, p):
    g = P.generate_ba(20000, 6, 3) if gen == "ba" else P.generate_rmat(15, 16, 1)
    P.device.bind_device(0)
    for part in P.partition_rows(g.num_nodes, p):
        want = numpy_structure(g, part)
        got = S._ShardStructure(g, part, P.device.current_device())
        nnz = got.nnz
        for name in ("row_ptr", "cols0", "col_ptr", "col_ent", "col_row", "order"):
            arr = getattr(got, name).cpu().numpy()
            if name in ("cols0", "col_ent", "col_row"):
                arr = arr[:nnz]
            if name == "order":
                arr = arr[:part.num_rows]
            assert np.array_equal(arr, want[name]), name
        assert got.n_hub == want["n_hub"]
        assert got.max_deg == want["max_deg"]
