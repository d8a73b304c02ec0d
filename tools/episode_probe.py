"""Time the device episode loop with and without CUDA-graph replay (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
from paper_2105_08764_b200.inference import DeviceEpisode
P.device.bind_device(0)
comm = P.WorkerGroup(1).comm(0)
params = P.PolicyParams.initialize(64, 5, seed=0)
for n in (1000, 20000):
    g = P.generate_ba(n, 4, 0)
    for use_graph in (False, True):
        for rep in range(2):
            st = P.PartitionedState([g], P.partition_rows(n, 1)[0])
            ep = DeviceEpisode(st, params, comm, P.SelectionSchedule.adaptive(), 8, use_graph=use_graph)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            chunks = 0; tcap = None
            while True:
                t1 = time.perf_counter()
                tp, ta, te, active = ep.run_chunk()
                if chunks == 1: tcap = time.perf_counter() - t1
                chunks += 1
                if not active.any(): break
            dt = time.perf_counter() - t0
            print(f"n={n} graph={use_graph} rep={rep} chunks={chunks} total {dt*1e3:.1f} ms "
                  f"per eval {dt/chunks/8*1e6:.0f} us  2nd chunk {tcap*1e3:.1f} ms captured={ep._graph is not None}", flush=True)
