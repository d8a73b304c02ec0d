"""Kernel breakdown of one BASELINE configs[3] training step (dev tool):
8 tuples of BA(2M,16), K=64, T=5, tau=4, through train_step."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
import bench
P.device.bind_device(0)
comm = P.WorkerGroup(1).comm(0)
ds = [P.generate_ba(2_000_000, 16, 0)]
part = P.partition_rows(ds[0].num_nodes, 1)[0]
buf = bench._train_buffer(P, ds, 8)
params = P.PolicyParams.initialize(64, 5, seed=0)
adam = P.AdamState.create(params, lr=1e-5)
cfg = P.TrainConfig(embed_dim=64, num_layers=5, batch_size=8, tau=4)
rng = np.random.default_rng(7)
for _ in range(2):
    P.train_step(buf, ds, params, adam, cfg, rng, comm, part)
torch.cuda.synchronize()
t0 = time.perf_counter()
P.train_step(buf, ds, params, adam, cfg, rng, comm, part)
torch.cuda.synchronize()
print(f"train step {(time.perf_counter() - t0) * 1e3:.2f} ms wall")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    P.train_step(buf, ds, params, adam, cfg, rng, comm, part)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=22, max_name_column_width=60))
