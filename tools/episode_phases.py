"""Walk a full adaptive episode exactly as solve() does (device loop, tail
chunking) and log progress every few seconds (dev tool): evaluations, active
rows, alive entries, ms per evaluation since the last line."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
from paper_2105_08764_b200.inference import DeviceEpisode
P.device.bind_device(0)
kind, scale, budget = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
# optional: evaluation counts at which to save the partial solution (packed
# bits) to gpurun_out/sol_<kind><scale>_<evals>.npy, for profiling later
# phases from a real mid-episode state
dumps = sorted(int(x) for x in sys.argv[4].split(",")) if len(sys.argv) > 4 else []
g = P.generate_rmat(scale, 16, 0) if kind == "rmat" else P.generate_ba(scale, 16, 0)
comm = P.WorkerGroup(1).comm(0)
params = P.PolicyParams.initialize(64, 5, seed=0)
start = os.environ.get("S2V_START_SOL")  # resume from a saved partial solution
sol = None if not start else np.unpackbits(np.load(start))[:g.num_nodes][None]
st = P.PartitionedState([g], P.partition_rows(g.num_nodes, 1)[0], solutions=sol)
ep = DeviceEpisode(st, params, comm, P.SelectionSchedule.adaptive(), 1, use_graph=False)
tail_rows = int(os.environ.get("S2V_TAIL_ROWS", "65536"))
tail = False
t0 = time.perf_counter()
last_t, last_e, evals = 0.0, 0, 0
active = np.array([True])
while active.any():
    if not tail and (ep.active_count() <= tail_rows or ep._mode[2]):
        ep.resize(16, use_graph=True)
        tail = True
        print("tail mode at eval", evals, flush=True)
    elif tail and not ep._mode[2] and ep.active_count() > tail_rows and ep.chunk != 1:
        ep.resize(1, use_graph=False)  # as solve(): the incremental trial fell back
        tail = False
        print("incremental trial fell back at eval", evals, flush=True)
    tp, ta, te, active = ep.run_chunk()
    evals += int(te.sum())
    while dumps and evals >= dumps[0]:
        np.save(f"gpurun_out/sol_{kind}{scale}_{dumps.pop(0)}.npy",
                np.packbits(st.sol_d.to("cpu").numpy()[:g.num_nodes]))
    now = time.perf_counter() - t0
    if now - last_t > 5 or not active.any() or now > budget or os.environ.get("S2V_VERBOSE"):
        d = int((tp[-1, 0] >= 0).sum())
        print(f"t {now:7.1f}s evals {evals:7d} active {ep.active_count():8d} alive "
              f"{int(st.residual_d.sum().item()):10d} d {d} "
              f"{(now - last_t) / max(evals - last_e, 1) * 1e3:.3f} ms/eval inc {int(ep._mode[2])} "
              f"overflow {int(ep.front_meta[2].item()) if ep.front is not None else -1} "
              f"fallbacks {ep.inc_fallbacks}", flush=True)
        last_t, last_e = now, evals
    if now > budget:
        break
