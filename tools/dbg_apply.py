import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
g = P.Graph(8, [(0, 2), (2, 4), (5, 7), (1, 6), (1, 3)])
sol = np.zeros((1, 8), np.uint8); sol[0, 2] = 1
def worker(comm):
    st = P.PartitionedState([g], P.partition_rows(8, 1)[0], solutions=sol)
    print("order", st.order.cpu().numpy(), "n_hub", st.n_hub)
    print("before cand", st.cand, "rdeg", st.rdeg.cpu().numpy())
    st.apply_action(5, slot=0)
    print("after cand", st.cand, "rdeg", st.rdeg.cpu().numpy(), "sol", st.sol, "res", st.local_residual)
P.run_workers(1, worker)
