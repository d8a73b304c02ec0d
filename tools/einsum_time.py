"""Per-launch time of s2v_theta2_einsum at the cfg4 shape (dev tool):
B = 8 slots x 2M rows, K = 64 fp32, CUDA events on the launching stream."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_08764_b200 as P
from paper_2105_08764_b200 import _lib
from paper_2105_08764_b200.device import stream_ptr

P.device.bind_device(0)
B, n, K = int(os.environ.get("AB_B", "8")), 2_000_000, 64
g = P.Graph(n, [(i, i + 1) for i in range(0, n - 1, 997)])


def worker(comm):
    st = P.PartitionedState([g] * B, P.partition_rows(n, 1)[0])
    lib = _lib.load()
    nb = lib.s2v_theta2_terms_bytes(_lib.S2V_F32, st.shard_ref(), K)
    t2c = torch.randn(nb // 4, device=st.device)
    tot = torch.empty(B * K, device=st.device)
    out = torch.empty(K, dtype=torch.float64, device=st.device)
    ms = []
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.call("s2v_theta2_einsum", _lib.S2V_F32, st.shard_ref(), K, t2c.data_ptr(),
                  tot.data_ptr(), out.data_ptr(), stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return ms


ms = P.run_workers(1, worker)[0][2:]
print(f"theta2_einsum B={B} rows={n}: median {np.median(ms):.3f} ms min {np.min(ms):.3f} ms")
