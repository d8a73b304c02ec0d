"""Walk an adaptive episode with the device loop and log how the residual
graph shrinks (dev tool): eval index, elapsed s, alive entries, candidates, d."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
from paper_2105_08764_b200.inference import DeviceEpisode
P.device.bind_device(0)
kind, scale, budget = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
g = P.generate_rmat(scale, 16, 0) if kind == "rmat" else P.generate_ba(scale, 16, 0)
comm = P.WorkerGroup(1).comm(0)
params = P.PolicyParams.initialize(64, 5, seed=0)
st = P.PartitionedState([g], P.partition_rows(g.num_nodes, 1)[0])
ep = DeviceEpisode(st, params, comm, P.SelectionSchedule.adaptive(), 1, use_graph=False)
t0 = time.perf_counter()
i = 0
last = 0
while True:
    tp, ta, te, active = ep.run_chunk()
    i += 1
    now = time.perf_counter() - t0
    if i % 100 == 0 or not active.any() or now > budget:
        res = int(st.residual_d.sum().item())
        cand = int(st.cand_d.sum().item())
        d = int((tp[0, 0] >= 0).sum())
        print(f"eval {i} t {now:.1f}s alive_entries {res} cand {cand} d {d} "
              f"dt/eval {(now - last) / 100 * 1e3:.2f} ms", flush=True)
        last = now
    if not active.any() or now > budget:
        break
