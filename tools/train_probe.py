"""Time the training step pieces at cfg2 / cfg4 sizes (dev tool)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2105_08764_b200 as P
from paper_2105_08764_b200 import agent

def run(name, dataset, B, tau, K=64, L=5):
    comm = P.WorkerGroup(1).comm(0)
    P.device.bind_device(0) if hasattr(P, "device") else None
    n = dataset[0].num_nodes
    part = P.partition_rows(n, 1)[0]
    rng = np.random.default_rng(0)
    buf = P.ReplayBuffer(1000)
    for i in range(B):
        gi = i % len(dataset)
        g = dataset[gi]
        bits = (rng.random(n) < 0.01).astype(np.uint8)
        st_deg = g.degrees()
        cands = np.flatnonzero((st_deg > 0) & (bits == 0))
        buf.add(P.ExperienceTuple(gi, P.pack_solution(bits), int(cands[rng.integers(len(cands))]), 0.0))
    params = P.PolicyParams.initialize(K, L, seed=0)
    adam = P.AdamState.create(params)
    cfg = P.TrainConfig(embed_dim=K, num_layers=L, batch_size=B, tau=tau)
    for it in range(3):
        torch.cuda.synchronize(); t0 = time.time()
        batch = buf.sample(np.random.default_rng(it), B)
        st = agent.tuples_to_graphs(batch, dataset, part)
        torch.cuda.synchronize(); t1 = time.time()
        tg = agent.batch_targets(batch, dataset, params, comm, part, 0.9).astype(np.float32)
        torch.cuda.synchronize(); t2 = time.time()
        acts = np.array([t.action for t in batch])
        tl = []
        for _ in range(tau):
            a = time.time()
            loss, grads = P.loss_and_gradients(st, acts, tg, params, comm)
            torch.cuda.synchronize(); b = time.time()
            P.adam_step(params, grads, adam)
            torch.cuda.synchronize(); c = time.time()
            tl.append((b - a, c - b))
        print(name, f"build {t1-t0:.3f} targets {t2-t1:.3f} iters", [f"{x:.3f}/{y:.4f}" for x, y in tl], f"total {time.time()-t0:.3f}", flush=True)

P.device.bind_device(0)
ds2 = [P.generate_ba(10000, 4, 100 + i) for i in range(32)]
run("cfg2 B=32 tau=4", ds2, 32, 4)
g = P.generate_ba(2_000_000, 16, 0)
run("cfg4 B=8 tau=4", [g], 8, 4)
