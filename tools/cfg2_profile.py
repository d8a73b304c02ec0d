"""Where a cfg2 train_step goes (dev tool): 32 x BA(10k,4), tau = 4, the
bench's buffer; device time per step (CUDA events) against the summed kernel
time of the same steps (torch.profiler), i.e. how much of the step is host
launch overhead rather than kernels."""
import os
import sys
import time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_08764_b200 as P
import bench

P.device.bind_device(0)
ds = [P.generate_ba(10_000, 4, 100 + i) for i in range(32)]
comm = P.WorkerGroup(1).comm(0)
part = P.partition_rows(ds[0].num_nodes, 1)[0]
buf = bench._train_buffer(P, ds, 32)
params = P.PolicyParams.initialize(64, 5, seed=0)
adam = P.AdamState.create(params, lr=1e-5)
cfg = P.TrainConfig(embed_dim=64, num_layers=5, batch_size=32, tau=4)
rng = np.random.default_rng(7)
for _ in range(3):
    P.train_step(buf, ds, params, adam, cfg, rng, comm, part)
torch.cuda.synchronize()
n = 5
t0 = time.perf_counter()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                        torch.profiler.ProfilerActivity.CPU]) as prof:
    for _ in range(n):
        P.train_step(buf, ds, params, adam, cfg, rng, comm, part)
    torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / n
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
kern = sum(e.device_time for e in ev) / n / 1e3
print(f"cfg2 step wall {wall*1e3:.2f} ms (under profiler), kernels {kern:.2f} ms, "
      f"{len(ev) // n} device events per step")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    P.train_step(buf, ds, params, adam, cfg, rng, comm, part)
e1.record()
torch.cuda.synchronize()
print(f"cfg2 step device time {e0.elapsed_time(e1) / n:.2f} ms (CUDA events, no profiler)")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18))
