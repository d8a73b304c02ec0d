"""Generate golden vectors by running the REFERENCE itself (this container only).

TEST INFRASTRUCTURE.  Imports the read-only reference package from
/root/reference/pkg/src and writes small fixtures under tests/golden/, which
travel to the GPU box (the reference does not).  Run:

    OPENBLAS_CORETYPE=SkylakeX python oracle/make_golden.py

OPENBLAS_CORETYPE=SkylakeX pins the sgemm kernel whose accumulation order the
fp32 contract describes.  Every fixture records the
reference call it came from.
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def _ref():
    sys.path.insert(0, str(REF))
    import graphrl  # noqa: E402
    return graphrl


def forward_fixture(R, name, n, m, seed, K, L, pseed, solfrac):
    g = R.generate_ba(n, m, seed)
    params = R.PolicyParams.initialize(K, L, seed=pseed)
    rng = np.random.default_rng(1234 + seed)
    sol = (rng.random(n) < solfrac).astype(np.uint8)
    comm = R.WorkerGroup(1).comm(0)
    st = R.PartitionedState([g], R.partition_rows(n, 1)[0], solutions=sol[None])
    emb = R.embed_forward(st, params, comm)                      # policy.py:182
    sc = R.q_forward(emb, st.cand, params, comm)                 # policy.py:214
    gsum = emb.sum(axis=2)[0]
    np.savez_compressed(OUT / f"{name}.npz", n=n, m=m, seed=seed, K=K, L=L, pseed=pseed,
                        sol=sol, h=np.ascontiguousarray(emb[0].T), scores=sc[0],
                        cand=st.cand[0], g=gsum, u1=(gsum[None] @ params.theta5.T)[0])


def solve_fixture(R, name, graphs, K, L, pseed, schedule=None):
    """Full solve with the per-evaluation picks recorded (select_top_d hook)."""
    import graphrl.inference as inf
    params = R.PolicyParams.initialize(K, L, seed=pseed)
    trace = []
    orig = inf.select_top_d

    def hooked(scores, cand, d):
        out = orig(scores, cand, d)
        trace.append(out)
        return out
    inf.select_top_d = hooked
    try:
        t0 = time.time()
        res = R.run_workers(1, lambda comm: R.solve(graphs, params, comm, schedule=schedule))[0]
        dt = time.time() - t0
    finally:
        inf.select_top_d = orig
    flat = np.concatenate([np.asarray(p, dtype=np.int64) for p in trace]) if trace else \
        np.zeros(0, np.int64)
    lens = np.array([len(p) for p in trace], dtype=np.int64)
    np.savez_compressed(
        OUT / f"{name}.npz", K=K, L=L, pseed=pseed,
        covers=np.concatenate([np.asarray(r.cover, dtype=np.int64) for r in res]),
        cover_lens=np.array([len(r.cover) for r in res]),
        evals=np.array([r.policy_evals for r in res]),
        skipped=np.array([r.skipped for r in res]),
        pick_flat=flat, pick_lens=lens, ref_seconds=dt)
    return dt


def train_fixture(R, name, n, m, B, K, L, tau, dtype=np.float32):
    """Reference training step pieces on a fixed sampled batch (agent.py:235-261)."""
    import graphrl.agent as ag
    dataset = [R.generate_ba(n, m, 100 + i) for i in range(B)]
    rng = np.random.default_rng(0)
    snaps, actions = [], []
    for g in dataset:
        bits = (rng.random(n) < 0.2).astype(np.uint8)
        st = R.PartitionedState([g], R.partition_rows(n, 1)[0], solutions=bits[None])
        cands = np.flatnonzero(st.cand[0])
        a = int(cands[int(rng.integers(len(cands)))])
        snaps.append(bits)
        actions.append(a)
    batch = [ag.ExperienceTuple(i, ag.pack_solution(snaps[i]), actions[i], 0.0)
             for i in range(B)]
    params = R.PolicyParams.initialize(K, L, seed=0, dtype=dtype)
    p0 = {k: v.copy() for k, v in params.as_dict().items()}
    adam = R.AdamState.create(params, lr=1e-5)
    comm = R.WorkerGroup(1).comm(0)
    part = R.partition_rows(n, 1)[0]
    state = ag.tuples_to_graphs(batch, dataset, part, dtype=params.dtype)
    targets = ag.batch_targets(batch, dataset, params, comm, part, 0.9).astype(params.dtype)
    losses, grads0 = [], None
    for it in range(tau):
        loss, grads = R.loss_and_gradients(state, np.array(actions), targets, params, comm)
        if it == 0:
            grads0 = grads
        R.adam_step(params, grads, adam)
        losses.append(loss)
    out = dict(n=n, m=m, B=B, K=K, L=L, tau=tau, snaps=np.stack(snaps),
               actions=np.array(actions), targets=targets, losses=np.array(losses))
    for k, v in p0.items():
        out[f"p0_{k}"] = v
    for k, v in grads0.items():
        out[f"g0_{k}"] = v
    for k, v in params.as_dict().items():
        out[f"p1_{k}"] = v
    for k in adam.m:
        out[f"m_{k}"] = adam.m[k]
        out[f"v_{k}"] = adam.v[k]
    np.savez_compressed(OUT / f"{name}.npz", **out)


def kat_fixture(R):
    """The reference's own dyadic known-answer vectors (pkg/tests/test_policy.py:16-42)."""
    sys.path.insert(0, "/root/reference/pkg/tests")
    import test_policy as tp  # noqa: E402
    data = {
        "source": "pkg/tests/test_policy.py:16-42",
        "HAND_THETA": {k: v.tolist() for k, v in tp.HAND_THETA.items()},
        "EXPECTED_PATH_L1": tp.EXPECTED_PATH_L1.tolist(),
        "EXPECTED_PATH_L2": tp.EXPECTED_PATH_L2.tolist(),
        "EXPECTED_PATH_SCORES": tp.EXPECTED_PATH_SCORES.tolist(),
        "EXPECTED_PATH_SCORES_EXTRACT": tp.EXPECTED_PATH_SCORES_EXTRACT.tolist(),
        "EXPECTED_CYCLE_L2": tp.EXPECTED_CYCLE_L2.tolist(),
        "EXPECTED_CYCLE_SCORES": tp.EXPECTED_CYCLE_SCORES.tolist(),
    }
    (OUT / "kat_dyadic.json").write_text(json.dumps(data, indent=1))


def generator_fixture(R):
    """SHA-256 of the reference generators' edge arrays (graphs.py:90-157),
    so the native generate_ba / numpy generate_er are pinned bit for bit."""
    import hashlib
    out = {"source": "graphrl.generate_ba / generate_er (pkg/src/graphrl/graphs.py:90-157)",
           "ba": [], "er": []}
    for n, d, seed in ((1000, 4, 0), (20000, 4, 3), (100000, 16, 0)):
        e = np.ascontiguousarray(R.generate_ba(n, d, seed).edge_array, dtype=np.int64)
        out["ba"].append({"n": n, "d": d, "seed": seed, "edges": int(e.shape[0]),
                          "sha256": hashlib.sha256(e.tobytes()).hexdigest()})
    for n, rho, seed in ((300, 0.05, 7), (5000, 0.002, 1)):
        e = np.ascontiguousarray(R.generate_er(n, rho, seed).edge_array, dtype=np.int64)
        out["er"].append({"n": n, "rho": rho, "seed": seed, "edges": int(e.shape[0]),
                          "sha256": hashlib.sha256(e.tobytes()).hexdigest()})
    (OUT / "generators.json").write_text(json.dumps(out, indent=1))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "gen":
        generator_fixture(_ref())
        return
    if len(sys.argv) > 1 and sys.argv[1] == "cfg2":
        # BASELINE configs[1]: 32 x BA(10000,4,seed=100+i), B=32, tau=4
        R = _ref()
        t0 = time.time()
        train_fixture(R, "train_cfg2_ba10k_b32_k64_l5", 10000, 4, 32, 64, 5, 4)
        print("cfg2", time.time() - t0)
        return
    if os.environ.get("OPENBLAS_CORETYPE") != "SkylakeX":
        print("warning: set OPENBLAS_CORETYPE=SkylakeX for the pinned sgemm order")
    OUT.mkdir(parents=True, exist_ok=True)
    R = _ref()
    kat_fixture(R)
    forward_fixture(R, "fwd_ba1000_k64_l5", 1000, 4, 0, 64, 5, 0, 0.0)
    forward_fixture(R, "fwd_ba1000_k64_l5_sol10", 1000, 4, 0, 64, 5, 0, 0.1)
    forward_fixture(R, "fwd_ba800_k32_l2", 800, 4, 1, 32, 2, 1, 0.05)
    forward_fixture(R, "fwd_ba5000_m8_k64_l5", 5000, 8, 3, 64, 5, 2, 0.2)
    print("solve ba1000", solve_fixture(R, "solve_ba1000_k64_l5", [R.generate_ba(1000, 4, 0)],
                                        64, 5, 0))
    print("solve ba1000 d1", solve_fixture(R, "solve_ba1000_k64_l5_single",
                                           [R.generate_ba(1000, 4, 0)], 64, 5, 0,
                                           R.SelectionSchedule.single()))
    print("solve batch3", solve_fixture(R, "solve_batch3_k32_l2",
                                        [R.generate_ba(800, 4, s) for s in (1, 2, 3)], 32, 2, 1))
    print("solve fixed8", solve_fixture(R, "solve_er300_fixed8_k16_l3",
                                        [R.generate_er(300, 0.05, 7)], 16, 3, 4,
                                        R.SelectionSchedule.fixed(8)))
    print("solve ba20000", solve_fixture(R, "solve_ba20000_k64_l5", [R.generate_ba(20000, 4, 0)],
                                         64, 5, 0))
    train_fixture(R, "train_ba1000_b4_k64_l5", 1000, 4, 4, 64, 5, 2)
    train_fixture(R, "train_ba600_b3_k16_l3_f64", 600, 4, 3, 16, 3, 2, dtype=np.float64)


if __name__ == "__main__":
    main()
