"""Host-side profile (cProfile) of the configs[1] training step (dev tool)."""
import cProfile, pstats, sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
import bench
P.device.bind_device(0)
comm = P.WorkerGroup(1).comm(0)
ds = [P.generate_ba(10000, 4, 100 + i) for i in range(32)]
part = P.partition_rows(10000, 1)[0]
buf = bench._train_buffer(P, ds, 32)
params = P.PolicyParams.initialize(64, 5, seed=0)
adam = P.AdamState.create(params, lr=1e-5)
cfg = P.TrainConfig(embed_dim=64, num_layers=5, batch_size=32, tau=4)
rng = np.random.default_rng(7)
for _ in range(3):
    P.train_step(buf, ds, params, adam, cfg, rng, comm, part)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    P.train_step(buf, ds, params, adam, cfg, rng, comm, part)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
