"""Where the bench's e2e step goes (dev tool): PartitionedState from a host
solution + solve_step, 10 steps, wall and device time; torch.profiler table."""
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


held = []


def step():
    while held:
        held.pop().release()
    st = P.PartitionedState([g], part, solutions=sol)
    held.append(st)
    picks, applied = solve_step(st, params, comm, sched, active)
    for v, a in zip(picks[0], applied[0]):
        if v >= 0 and a:
            sol[0, v] = 1


for _ in range(3):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    step()
torch.cuda.synchronize()
print(f"e2e step {(time.perf_counter() - t0) / 10 * 1e3:.2f} ms wall")
t0 = time.perf_counter()
st = P.PartitionedState([g], part, solutions=sol)
torch.cuda.synchronize()
print(f"state build {(time.perf_counter() - t0) * 1e3:.2f} ms")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="self_cpu_time_total", row_limit=25,
                                max_name_column_width=50))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15, max_name_column_width=50))
