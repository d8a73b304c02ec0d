"""Per-step wall times of the bench's e2e loop (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
from paper_2105_08764_b200.inference import solve_step
P.device.bind_device(0)
g = P.generate_ba(2_000_000, 16, 0)
comm = P.WorkerGroup(1).comm(0)
params = P.PolicyParams.initialize(64, 5, seed=0)
part = P.partition_rows(g.num_nodes, 1)[0]
sched = P.SelectionSchedule.adaptive()
sol = np.zeros((1, g.num_nodes), np.uint8)
active = np.array([True])
times = []
for i in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = P.PartitionedState([g], part, solutions=sol)
    t1 = time.perf_counter()
    picks, applied = solve_step(st, params, comm, sched, active)
    for v, a in zip(picks[0], applied[0]):
        if v >= 0 and a:
            sol[0, v] = 1
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    times.append((t1 - t0, t2 - t1))
for i, (a, b) in enumerate(times):
    print(f"step {i:2d} state {a*1e3:6.2f} ms  solve_step {b*1e3:6.2f} ms")
