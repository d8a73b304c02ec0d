"""cfg4 full-size gradients: GPU fp32 and the reference's fp32 against a GPU
fp64 evaluation of the same step (dev tool for the tolerance analysis)."""
import json, sys
import numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2105_08764_b200 as P
from reference_math import scale_error
gold = json.load(open("/root/repo/tests/golden/full_cfg4_train.json"))
g = P.generate_ba(2_000_000, 16, 0)
n = g.num_nodes
snaps = np.zeros((2, n), np.uint8); snaps[1, gold["snap1"]] = 1
batch = [P.ExperienceTuple(0, P.pack_solution(snaps[i]), gold["actions"][i], 0.0) for i in range(2)]
targets = np.asarray(gold["targets"], np.float32)
out = {}
for dt in (np.float32, np.float64):
    params = P.PolicyParams.initialize(64, 5, seed=0).astype(dt)
    def worker(comm):
        part = P.partition_rows(n, 1)[0]
        st = P.tuples_to_graphs(batch, [g], part, dtype=dt)
        return P.loss_and_gradients(st, np.array(gold["actions"]), targets.astype(dt), params, comm)
    out[dt] = P.run_workers(1, worker)[0]
ref = {k: np.asarray(v) for k, v in gold["grads"].items()}
l64, g64 = out[np.float64]
l32, g32 = out[np.float32]
print("loss ref", gold["loss"], "gpu32", l32, "gpu64", l64)
for k in P.PARAM_NAMES:
    print(k, "gpu32 vs f64 %.2e" % scale_error(g32[k], g64[k]).max(),
          "ref32 vs f64 %.2e" % scale_error(ref[k], g64[k]).max(),
          "gpu32 vs ref %.2e" % scale_error(g32[k], ref[k]).max())
