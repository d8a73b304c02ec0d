"""A/B timing of the cfg3 inference step (dev tool): BA(2M,16), K = 64,
solve_step from S = {} on one resident state, CUDA events per step.  Run one
process per setting of an env knob, e.g.
    for mb in 32 48 64; do S2V_HOT_MB=$mb python tools/round_ab.py; done"""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2105_08764_b200 as P
from paper_2105_08764_b200.inference import solve_step

P.device.bind_device(0)
g = P.generate_ba(2_000_000, 16, 0)
comm = P.WorkerGroup(1).comm(0)
params = P.PolicyParams.initialize(64, 5, seed=0)
part = P.partition_rows(g.num_nodes, 1)[0]
sched = P.SelectionSchedule.adaptive()
active = np.array([True])


def worker(comm):
    st = P.PartitionedState([g], part)
    ms = []
    for i in range(int(os.environ.get("AB_STEPS", "24"))):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        solve_step(st, params, comm, sched, active)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    return ms


ms = P.run_workers(1, worker)[0][4:]
knobs = {k: v for k, v in os.environ.items() if k.startswith("S2V_")}
print(f"AB {knobs} step ms: median {np.median(ms):.3f} min {np.min(ms):.3f} "
      f"mean {np.mean(ms):.3f}")
