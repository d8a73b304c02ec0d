import numpy as np, sys
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
g = P.generate_ba(500, 5, 3)
params = P.PolicyParams.initialize(16, 4, seed=3, dtype=np.float64)
def worker(comm):
    part = P.partition_rows(g.num_nodes, 1)[0]
    st = P.PartitionedState([g], part, dtype=params.dtype)
    emb = P.embed_forward(st, params, comm)
    h = np.asarray(emb)
    print("embed ok", h.shape)
    sc = P.q_forward(emb, st.cand, params, comm)
    print("scores ok")
P.run_workers(1, worker)
