"""One cfg4-style loss_and_gradients (B tuples of BA(2M,16)) for profiling."""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
P.device.bind_device(0)
g = P.generate_ba(2_000_000, 16, 0)
n = g.num_nodes
rng = np.random.default_rng(0)
sols = (rng.random((B, n)) < 0.01).astype(np.uint8)
comm = P.WorkerGroup(1).comm(0)
st = P.PartitionedState([g] * B, P.partition_rows(n, 1)[0], solutions=sols)
cand = st.cand
acts = np.array([int(np.flatnonzero(cand[b])[5]) for b in range(B)])
params = P.PolicyParams.initialize(64, 5, seed=0)
for _ in range(2):
    loss, grads = P.loss_and_gradients(st, acts, np.full(B, -1.0, np.float32), params, comm)
torch.cuda.synchronize()
print("loss", loss)
