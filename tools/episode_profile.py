"""Kernel time breakdown of device-episode evaluations mid-episode (dev
tool): walk `skip` evaluations, then profile `n` with torch.profiler (CUPTI)."""
import sys, time
import torch
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
from paper_2105_08764_b200.inference import DeviceEpisode
P.device.bind_device(0)
kind, scale, skip, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
chunk = int(sys.argv[5]) if len(sys.argv) > 5 else 1
solfrac = float(sys.argv[6]) if len(sys.argv) > 6 else 0.0
g = P.generate_rmat(scale, 16, 0) if kind == "rmat" else P.generate_ba(scale, 16, 0)
comm = P.WorkerGroup(1).comm(0)
params = P.PolicyParams.initialize(64, 5, seed=0)
import numpy as np
if len(sys.argv) > 7:  # a saved mid-episode solution (tools/episode_phases.py)
    sol = np.unpackbits(np.load(sys.argv[7]))[:g.num_nodes][None]
else:
    sol = (np.random.default_rng(0).random(g.num_nodes) < solfrac).astype(np.uint8)[None]
st = P.PartitionedState([g], P.partition_rows(g.num_nodes, 1)[0], solutions=sol)
ep = DeviceEpisode(st, params, comm, P.SelectionSchedule.adaptive(), chunk,
                   use_graph=chunk > 1)
for _ in range(skip // chunk):
    ep.run_chunk()
torch.cuda.synchronize()
print("active rows", ep.active_count(), "alive entries", int(st.residual_d.sum().item()))
t0 = time.perf_counter()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(n // chunk):
        ep.run_chunk()
    torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{n} evals, {dt / n * 1e3:.3f} ms/eval wall (profiled)")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=60))
