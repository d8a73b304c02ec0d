"""Full-size golden checksums from the REFERENCE itself (BASELINE cfg3/cfg4).

TEST INFRASTRUCTURE.  The arrays at BA(2M,16) are too large to commit
(512 MB per embedding), so this records SHA-256 digests of the reference's
fp32 bytes plus small vectors (g, u1, the first steps' picks, losses and
gradients).  The graph is the reference's generate_ba(2_000_000, 16, 0); to
avoid its 216 s pure-Python generation the bit-identical native generator's
edge list is fed to the reference's own Graph (tests/test_oracle.py pins
the generator against the reference at smaller sizes).  Run here only:

    OPENBLAS_CORETYPE=SkylakeX python oracle/make_golden_full.py [infer|mid|train]

`mid` is SURVEY.md 8(d)'s mid-episode cfg3 state: S_mid = a seeded random
35% of the nodes (default_rng(11)), built on both sides with
PartitionedState(..., solutions=S_mid), then one forward and the first
adaptive steps from it.
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden"


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(which: str):
    sys.path.insert(0, str(ROOT))
    import paper_2105_08764_b200 as P
    sys.path.insert(0, "/root/reference/pkg/src")
    import graphrl as R
    import graphrl.inference as inf
    t0 = time.time()
    mine = P.generate_ba(2_000_000, 16, 0)
    g = R.Graph(2_000_000, mine.edge_array)
    print("graph", g.num_edges, f"{time.time() - t0:.1f}s", flush=True)
    params = R.PolicyParams.initialize(64, 5, seed=0)
    comm = R.WorkerGroup(1).comm(0)
    part = R.partition_rows(g.num_nodes, 1)[0]
    sol = None
    if which == "mid":
        sol = (np.random.default_rng(11).random(g.num_nodes) < 0.35).astype(np.uint8)[None]
    if which in ("infer", "mid"):
        st = R.PartitionedState([g], part, solutions=sol)
        t0 = time.time()
        emb = R.embed_forward(st, params, comm)
        sc = R.q_forward(emb, st.cand, params, comm)
        gsum = emb.sum(axis=2)[0]
        u1 = (gsum[None] @ params.theta5.T)[0]
        h = np.ascontiguousarray(emb[0].T)
        print("forward", f"{time.time() - t0:.1f}s", flush=True)
        out = {"config": "BA(2000000,16,0), K=64, L=5, params seed 0, " + (
                   "S = {}" if sol is None else
                   "S_mid = default_rng(11).random(N) < 0.35 (%d nodes)" % int(sol.sum())),
               "residual": int(st.local_residual[0]),
               "h_sha256": digest(h), "scores_sha256": digest(sc[0]),
               "cand_sha256": digest(st.cand[0]), "g": gsum.tolist(), "u1": u1.tolist(),
               "h_row0": h[0].tolist(), "scores_head": sc[0][:16].tolist()}
        # first adaptive steps of _solve_batch (inference.py:107-147)
        picks_log = []
        orig = inf.select_top_d

        def hooked(scores, cand, d):
            res = orig(scores, cand, d)
            picks_log.append(res)
            return res
        inf.select_top_d = hooked
        try:
            st2 = R.PartitionedState([g], part, solutions=sol)
            sched = R.SelectionSchedule.adaptive()
            for _ in range(3 if sol is None else 2):
                t0 = time.time()
                e = R.embed_forward(st2, params, comm)
                s2 = R.q_forward(e, st2.cand, params, comm)
                gl = comm.all_gather(R.masked_scores(s2, st2.cand), axis=-1)
                cm = np.isfinite(gl[0])
                picks = inf.select_top_d(gl[0], cm, sched.d_for(int(cm.sum()), g.num_nodes))
                applied = []
                for j, v in enumerate(picks):
                    if j > 0 and not st2.cand[0, v]:
                        continue
                    st2.apply_action(v, 0)
                    applied.append(v)
                print("step", picks, f"{time.time() - t0:.1f}s", flush=True)
        finally:
            inf.select_top_d = orig
        out["first_steps_picks"] = picks_log
        (OUT / ("full_cfg3_infer.json" if sol is None else "full_cfg3_mid.json")).write_text(
            json.dumps(out))
    else:
        # cfg4 at the CPU oracle's size: B=2 tuples, tau=1
        import graphrl.agent as ag
        snaps = np.zeros((2, g.num_nodes), np.uint8)
        for v in (4, 3, 15, 0, 17, 12, 9, 16):
            snaps[1, v] = 1
        actions = [4, 5]
        batch = [ag.ExperienceTuple(0, ag.pack_solution(snaps[i]), actions[i], 0.0)
                 for i in range(2)]
        t0 = time.time()
        state = ag.tuples_to_graphs(batch, [g], part)
        targets = ag.batch_targets(batch, [g], params, comm, part, 0.9).astype(np.float32)
        print("targets", targets, f"{time.time() - t0:.1f}s", flush=True)
        loss, grads = R.loss_and_gradients(state, np.array(actions), targets, params, comm)
        print("loss", loss, f"{time.time() - t0:.1f}s", flush=True)
        out = {"config": "BA(2000000,16,0), K=64, L=5, B=2 tuples (S={} and S={4,3,15,0,17,12,9,16}),"
                         " actions [4,5], gamma 0.9",
               "snap1": [4, 3, 15, 0, 17, 12, 9, 16], "actions": actions,
               "targets": targets.tolist(), "loss": loss,
               "grads": {k: v.tolist() for k, v in grads.items()}}
        (OUT / "full_cfg4_train.json").write_text(json.dumps(out))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "infer")
