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


ALG5 = dict(n=400, m=4, graphs=4, seed0=200, K=64, L=3, B=4, tau=2, lr=1e-4, eps_start=1.0,
            eps_end=0.0, eps_decay=12, capacity=64, cfg_seed=5, eval_every=10, steps=40,
            resume_at=20, eval_n=400, eval_seed=999, ref_size=200)


def alg5_fixture(R):
    """Algorithm 5 end to end: the reference's train() (agent.py:273-348)
    for ALG5["steps"] steps on a BA dataset, with every act / compute_target
    / train_step result recorded (hooks on the agent module), plus the same
    run split in two with the checkpoint + train_state.npz resume of
    cli.py:152-178 (params via save/load_checkpoint, Adam m/v/step/lr and
    global_step via np.savez)."""
    import tempfile
    import graphrl.agent as ag
    c = ALG5
    dataset = [R.generate_ba(c["n"], c["m"], c["seed0"] + i) for i in range(c["graphs"])]
    evals = [R.generate_ba(c["eval_n"], c["m"], c["eval_seed"])]
    cfg = ag.TrainConfig(embed_dim=c["K"], num_layers=c["L"], batch_size=c["B"], tau=c["tau"],
                         learning_rate=c["lr"], replay_capacity=c["capacity"],
                         eps_start=c["eps_start"], eps_end=c["eps_end"],
                         eps_decay_steps=c["eps_decay"], eval_every=c["eval_every"],
                         seed=c["cfg_seed"])
    log = {"act": [], "target": [], "loss": []}
    o_act, o_tgt, o_ts = ag.act, ag.compute_target, ag.train_step

    def h_act(*a, **k):
        v = o_act(*a, **k)
        log["act"].append(int(v))
        return v

    def h_tgt(*a, **k):
        t = o_tgt(*a, **k)
        log["target"].append(float(t))
        return t

    def h_ts(*a, **k):
        ls = o_ts(*a, **k)
        log["loss"].append([float(x) for x in ls])
        return ls
    ag.act, ag.compute_target, ag.train_step = h_act, h_tgt, h_ts
    out = {}
    try:
        def run(tag, **kw):
            for key in log:
                log[key] = []
            probe = {}
            params, metrics = R.run_workers(1, lambda comm: ag.train(
                dataset, cfg, comm, eval_graphs=evals, reference_sizes=[c["ref_size"]],
                probe=probe, **kw))[0]
            out[f"{tag}_act"] = np.array(log["act"], np.int64)
            out[f"{tag}_target"] = np.array(log["target"], np.float64)
            flat = [x for ls in log["loss"] for x in ls]
            out[f"{tag}_loss"] = np.array(flat, np.float64)
            out[f"{tag}_loss_len"] = np.array([len(ls) for ls in log["loss"]], np.int64)
            out[f"{tag}_metrics"] = np.array([[r.step, r.epsilon, r.loss, r.mean_approx_ratio,
                                               r.cover_size_mean] for r in metrics], np.float64)
            adam = probe["adam_state"]
            for k, v in params.as_dict().items():
                out[f"{tag}_p_{k}"] = v
                out[f"{tag}_m_{k}"] = adam.m[k]
                out[f"{tag}_v_{k}"] = adam.v[k]
            out[f"{tag}_adam_step"] = np.array(adam.step)
            out[f"{tag}_global_step"] = np.array(probe["global_step"])
            return params, adam, probe
        run("full", max_steps=c["steps"])
        params, adam, probe = run("first", max_steps=c["resume_at"])
        with tempfile.TemporaryDirectory() as d:   # cli.py:152-178 round trip
            R.save_checkpoint(params, Path(d) / "checkpoint.bin")
            arrays = {"global_step": probe["global_step"], "adam_step": adam.step, "lr": adam.lr}
            for name, arr in adam.m.items():
                arrays[f"m_{name}"] = arr
            for name, arr in adam.v.items():
                arrays[f"v_{name}"] = arr
            np.savez(Path(d) / "train_state.npz", **arrays)
            p2 = R.load_checkpoint(Path(d) / "checkpoint.bin")
            blob = np.load(Path(d) / "train_state.npz")
            a2 = R.AdamState(m={k: blob[f"m_{k}"] for k in p2.as_dict()},
                             v={k: blob[f"v_{k}"] for k in p2.as_dict()},
                             step=int(blob["adam_step"]), lr=float(blob["lr"]))
            run("resumed", max_steps=c["steps"] - c["resume_at"], params=p2, adam=a2,
                start_step=int(blob["global_step"]))
    finally:
        ag.act, ag.compute_target, ag.train_step = o_act, o_tgt, o_ts
    np.savez_compressed(OUT / "alg5_train_ba400_k64_l3.npz", **out)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "alg5":
        t0 = time.time()
        alg5_fixture(_ref())
        print("alg5", time.time() - t0)
        return
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
