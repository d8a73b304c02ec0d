#!/usr/bin/env python
"""Benchmark: one MVC structure2vec-DQN inference step on the >30M-edge
Barabasi-Albert graph (BASELINE.json configs[2]: BA(2M, 16), K=64, T=5),
node-sharded over N GPUs (one process per GPU under torchrun).

A step = one policy evaluation (5 embedding rounds, pairwise global sum, Q
scores, adaptive top-d keys) + selection + group apply -- one iteration of
the reference's _solve_batch loop (pkg/src/graphrl/inference.py:107-147).
Consecutive steps walk the episode from S = {} (the state evolves as in a
real solve).  `value` is device time per step with the graph resident in HBM;
`e2e` rebuilds the state from a host solution vector each step (H2D inside
the timed region) through the public PartitionedState + solve_step API.

--impl reference times the reference algorithm's CPU implementation
(oracle/port.py: the reference's numpy/scipy calls, restated) on the host.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RL inference step time on 30M-edge BA graph (s)"
MEASURED = ROOT / "MEASURED_PEAKS.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nodes", type=int, default=2_000_000)
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-train", action="store_true")
    ap.add_argument("--train-steps", type=int, default=5)
    ap.add_argument("--no-extra", action="store_true", help="skip the cfg1 / cfg5 legs")
    ap.add_argument("--rmat-scale", type=int, default=22)
    ap.add_argument("--full-episode", action="store_true",
                    help="also time a full adaptive solve of the R-MAT graph (configs[4]); "
                         "takes minutes")
    ap.add_argument("--same-device", action="store_true",
                    help="bind every rank to cuda:0 (multi-process test on one GPU)")
    return ap.parse_args()


def workload(args):
    return {"workload": f"MVC inference step, BA({args.nodes},{args.m},seed=0), K=64, T=5, "
                        f"adaptive 8/4/2/1, node-sharded",
            "graph": f"generate_ba({args.nodes}, {args.m}, 0)", "embed_dim": 64, "rounds": 5,
            "l2": "inputs larger than L2 (512 MB embedding buffers, 256 MB CSR)",
            "parallelism": f"node-rows x{args.gpus}"}


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region: NVML
    every 10 ms (a query costs microseconds), else nvidia-smi every 0.2 s."""
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, {reason flags})
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self.source = "nvml"

    def _nvml_open(self):
        """NVML handle opened before the timed region (init takes ~0.1 s)."""
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            self._nv = (pynvml, h, bits, mx)
        except Exception:
            self._nv = None

    def _nvml_sample(self):
        pynvml, h, bits, mx = self._nv
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.rows.append((float(sm), mx, {n for n, b in bits.items() if r & b}))

    def _nvml(self):
        while not self._stop.is_set():
            self._nvml_sample()
            self._stop.wait(0.01)

    def _smi(self):
        fields = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" +
                                      fields, "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                r = [x.strip() for x in out.split(",")]
                if len(r) >= 6 and r[0].replace(".", "").isdigit():
                    self.rows.append((float(r[0]), float(r[1]),
                                      {n for i, n in enumerate(self.NAMES)
                                       if r[2 + i].lower().startswith("active")}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            if self._nv is None:
                raise RuntimeError("no NVML")
            self._nvml()
        except Exception:
            self.source = "nvidia-smi"
            self._smi()

    def __enter__(self):
        self._nvml_open()
        self._t.start()
        return self

    def __exit__(self, *exc):
        if self._nv is not None:  # one sample at the end of the timed region too
            try:
                self._nvml_sample()
            except Exception:
                pass
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])),
                "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted(set().union(*[r[2] for r in self.rows])),
                "samples": len(self.rows), "source": self.source}


def peaks():
    """HBM peak (GB/s) for the roofline: MEASURED_PEAKS.json (driver-written;
    the round kernel is timed inside a step, so a 'sustained' HBM figure is
    preferred over a burst one), else the B200_PROFILING.md fallback."""
    try:
        d = json.loads(MEASURED.read_text())
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"
    flat = {}

    def walk(x, path):
        if isinstance(x, dict):
            for k, v in x.items():
                walk(v, f"{path}.{k}" if path else str(k))
        elif isinstance(x, (int, float)) and not isinstance(x, bool):
            flat[path.lower()] = float(x)
    walk(d, "")
    hbm = {k: v for k, v in flat.items()
           if ("hbm" in k or "copy" in k or "dram" in k) and "tf" not in k and v > 0}
    for pick in ([k for k in hbm if "sustain" in k], [k for k in hbm if "burst" not in k],
                 list(hbm)):
        if pick:
            k = sorted(pick)[0]
            v = hbm[k]
            return (v * 1000.0 if v < 100 else v), f"measured (MEASURED_PEAKS.json {k})"
    return 6650.0, "fallback (B200_PROFILING.md; no HBM key in MEASURED_PEAKS.json)"


# ---------------------------------------------------------------------------
# reference CPU arm / cpu_baseline
# ---------------------------------------------------------------------------


def cpu_state(graph):
    from oracle import port
    t0 = time.perf_counter()
    st = port.ResidualState([graph.edge_array], graph.num_nodes, dtype=np.float32)
    return st, time.perf_counter() - t0


def cpu_sample(st, theta, layers=5):
    """One bounded sample of the reference algorithm's inference step on the
    same graph: one full embedding round (spmm + theta4 + relu) timed, times
    the 5 rounds of a step, plus q_forward + masked select + group apply.
    Returns (estimated step seconds, detail)."""
    from oracle import port
    t0 = time.perf_counter()
    h1 = port.embed(st, theta, 1)
    t_round = time.perf_counter() - t0
    t0 = time.perf_counter()
    s = port.scores(h1, st.cand, theta)
    gl = port.masked(s, st.cand)
    cm = np.isfinite(gl[0])
    picks = port.select_top_d(gl[0], cm, port.d_for(int(cm.sum()), st.n))
    for j, v in enumerate(picks):
        if j > 0 and not st.cand[0, v]:
            continue
        st.apply(v, 0)
    t_rest = time.perf_counter() - t0
    est = layers * t_round + t_rest
    return est, {"round_s": round(t_round, 3), "q_select_apply_s": round(t_rest, 3)}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2105_08764_b200.graphs as G
    from paper_2105_08764_b200.policy import PolicyParams
    graph = G.generate_ba(args.nodes, args.m, 0)
    theta = PolicyParams.initialize(64, 5, seed=0).as_dict()
    cores = os.cpu_count()
    st, build = cpu_state(graph)
    for _ in range(args.warmup):
        cpu_sample(st, theta)
    vals, detail = [], None
    for _ in range(args.steps):
        v, detail = cpu_sample(st, theta)
        vals.append(v)
    value = float(np.mean(vals))
    sample = ("reference algorithm (oracle/port.py, numpy/scipy restatement of graphrl) "
              "on the same graph: per step, 1 timed embedding round x 5 + q_forward + "
              f"select + apply; {detail}; state build {build:.1f}s excluded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": workload(args),
            "cpu_baseline": {"value": value, "unit": "s", "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# training-step legs (BASELINE configs[1] and configs[3])
# ---------------------------------------------------------------------------


def _train_buffer(P, dataset, B, seed=0, frac=0.01):
    """B replay tuples (one per batch slot): snapshot ~ Bernoulli(frac), action
    a uniformly drawn candidate."""
    rng = np.random.default_rng(seed)
    buf = P.ReplayBuffer(max(B, 1))
    for i in range(B):
        gi = i % len(dataset)
        g = dataset[gi]
        bits = (rng.random(g.num_nodes) < frac).astype(np.uint8)
        rp, cols = g.csr_arrays()
        deg = np.diff(rp)
        cands = np.flatnonzero((deg > 0) & (bits == 0))
        buf.add(P.ExperienceTuple(gi, P.pack_solution(bits), int(cands[rng.integers(len(cands))]),
                                  0.0))
    return buf


def train_leg(P, comm, dataset, B, tau, steps, warmup, name):
    """Time train_step (public API: sample, tuples_to_graphs, batch_targets,
    tau x (loss_and_gradients + adam_step)) with CUDA events."""
    import torch
    n = dataset[0].num_nodes
    part = P.partition_rows(n, comm.size)[comm.rank]
    buf = _train_buffer(P, dataset, B)
    params = P.PolicyParams.initialize(64, 5, seed=0)
    adam = P.AdamState.create(params, lr=1e-5)
    cfg = P.TrainConfig(embed_dim=64, num_layers=5, batch_size=B, tau=tau)
    rng = np.random.default_rng(7)
    for _ in range(warmup):
        P.train_step(buf, dataset, params, adam, cfg, rng, comm, part)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    losses = []
    for _ in range(steps):
        losses = P.train_step(buf, dataset, params, adam, cfg, rng, comm, part)
    e1.record()
    torch.cuda.synchronize()
    return {"workload": name, "value": e0.elapsed_time(e1) / steps / 1e3, "unit": "s",
            "B": B, "tau": tau, "steps": steps, "warmup": warmup,
            "last_losses": [float(x) for x in losses],
            "path": "train_step(buffer, dataset, params, adam, cfg, rng, comm, part)"}


def cpu_train_sample(dataset, B_sample, B, tau):
    """Reference algorithm (oracle/port.py) training step on B_sample of the B
    tuples, scaled by B / B_sample (the step is linear in B)."""
    from oracle import port
    import paper_2105_08764_b200 as P
    n = dataset[0].num_nodes
    buf = _train_buffer(P, dataset, B)
    tuples = [buf[i] for i in range(B_sample)]
    theta = P.PolicyParams.initialize(64, 5, seed=0).as_dict()
    edges = [dataset[t.graph_index].edge_array for t in tuples]
    snaps = np.stack([P.unpack_solution(t.solution_snapshot, n) for t in tuples])
    acts = np.array([t.action for t in tuples])
    t0 = time.perf_counter()
    st = port.ResidualState(edges, n, solutions=snaps)
    tg = port.batch_targets(edges, n, snaps, acts, theta, 5, 0.9).astype(np.float32)
    m = {k: np.zeros_like(v) for k, v in theta.items()}
    v = {k: np.zeros_like(x) for k, x in theta.items()}
    step = 0
    for _ in range(tau):
        _, grads = port.loss_and_grads(st, acts, tg, theta, 5)
        step = port.adam(theta, grads, m, v, step, 1e-5)
    dt = time.perf_counter() - t0
    return {"value": dt * B / B_sample, "unit": "s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle/port.py train step on {B_sample} of {B} tuples (tuples_to_graphs + "
                      f"batch_targets + {tau} x (loss_and_grads + adam)) = {dt:.2f}s, "
                      f"scaled x{B / B_sample:g}"}


# ---------------------------------------------------------------------------
# other inference configs: cfg1 (launch-bound small graph) and cfg5 (R-MAT)
# ---------------------------------------------------------------------------


def make_stepper(P, state, params, comm, sched):
    """One inference step exactly as solve() runs it: the device-resident loop
    (DeviceEpisode, one evaluation per read-back) at P = 1, else solve_step."""
    from paper_2105_08764_b200.inference import DeviceEpisode, _device_loop_ok, solve_step
    if _device_loop_ok(state, params, comm, sched):
        ep = DeviceEpisode(state, params, comm, sched, 1, use_graph=False)
        return (lambda: ep.run_chunk()), "device episode loop (inference.DeviceEpisode)"
    active = np.array([True] * state.batch)
    return (lambda: solve_step(state, params, comm, sched, active)), "inference.solve_step"


def infer_leg(P, comm, graph, steps, warmup, name):
    """Device time per inference step (solve_step) walking an episode from
    S = {}; stops early if the episode ends."""
    import torch
    from paper_2105_08764_b200.inference import solve_step
    part = P.partition_rows(graph.num_nodes, comm.size)[comm.rank]
    params = P.PolicyParams.initialize(64, 5, seed=0)
    sched = P.SelectionSchedule.adaptive()
    state = P.PartitionedState([graph], part)
    step, path = make_stepper(P, state, params, comm, sched)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    done = 0
    for _ in range(steps):
        if int(state.local_residual.sum()) == 0:
            break
        step()
        done += 1
    e1.record()
    torch.cuda.synchronize()
    rp, _ = graph.csr_arrays()
    deg = np.diff(rp)
    return {"workload": name, "value": e0.elapsed_time(e1) / max(done, 1) / 1e3, "unit": "s",
            "steps": done, "warmup": warmup, "nodes": graph.num_nodes, "path": path,
            "edges": graph.num_edges, "max_degree": int(deg.max()),
            "hub_rows": int(state.n_hub), "isolated_frac": float(np.mean(deg == 0))}


def full_solve_leg(P, comm, graph):
    import torch
    params = P.PolicyParams.initialize(64, 5, seed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    (res,) = P.solve([graph], params, comm)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, res


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import paper_2105_08764_b200 as P
    from paper_2105_08764_b200 import _lib, policy
    from paper_2105_08764_b200.device import bind_device
    from paper_2105_08764_b200.inference import solve_step

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # --same-device: every rank on cuda:0 (exercises the multi-process path on
    # a one-GPU box); otherwise one GPU per rank
    bind_device(0 if args.same_device else local)
    if world > 1:
        import torch.distributed as dist
        # host-side plumbing only (barrier, timing max, small host exchanges);
        # the halo data path is the IPC peer-memory transport (DistComm)
        dist.init_process_group("gloo")
        comm = P.DistComm()
    else:
        comm = P.WorkerGroup(1).comm(0)

    def barrier():
        if world > 1:
            torch.cuda.synchronize()
            comm.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        return float(max(comm.all_gather(np.array([x], np.float64), tag="bench")))

    t0 = time.time()
    graph = P.generate_ba(args.nodes, args.m, 0)
    graph.csr_arrays()
    t_gen = time.time() - t0
    params = P.PolicyParams.initialize(64, 5, seed=0)
    part = P.partition_rows(graph.num_nodes, world)[rank]
    sched = P.SelectionSchedule.adaptive()
    active = np.array([True])
    t0 = time.time()
    state = P.PartitionedState([graph], part)
    torch.cuda.synchronize()
    t_state = time.time() - t0

    step, step_path = make_stepper(P, state, params, comm, sched)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    launches0 = _lib.launch_count
    alive_entries = int(state.local_residual.sum())
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    step_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    launches = _lib.launch_count - launches0

    # roofline of the dominant kernel (the fused embedding round): per-launch
    # CUDA events on the launching stream over one more step
    policy.ROUND_TIMER = []
    alive_now = int(state.local_residual.sum())
    step()
    torch.cuda.synchronize()
    rounds = policy.ROUND_TIMER
    policy.ROUND_TIMER = None
    round_ms = float(np.mean([a.elapsed_time(b) for a, b in rounds]))
    rows = part.num_rows
    nnz_loc = state.nnz
    algo_bytes = 8 * (rows + 1) + 4 * nnz_loc + 256 * alive_now + 256 * rows + 4 * rows + rows
    peak, peak_src = peaks()
    achieved = algo_bytes / (round_ms * 1e-3) / 1e9
    traffic = None
    try:  # DRAM bytes per launch from the committed ncu --set full capture
        tr = json.loads((ROOT / "profiles" / "r1_round64_traffic.json").read_text())
        if args.nodes == 2_000_000 and args.m == 16 and world == 1:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_source": "profiles/r1_round64_traffic.json (ncu dram__bytes_read+write)",
                "kernel": "round64_kernel (fused gather-SpMM + theta4 FMA chain + e12 + relu), "
                          "rounds 3..5 (round 2 gathers the per-degree h1 table, round 1 is "
                          "skipped)",
                "round_ms": round(round_ms, 4), "algorithmic_bytes_per_launch": algo_bytes,
                "peak_source": peak_src,
                "bytes_model": "8(rows+1) row_ptr + 4 nnz cols + 256 alive gathers + 256 rows h_out"
                               " + 4 rows rdeg + rows sol"}

    # end to end through the public API: host solution vector -> state -> step
    e2e = None
    if not args.no_e2e:
        sol_host = np.zeros((1, graph.num_nodes), dtype=np.uint8)
        sol_host[0, part.row_start:part.row_stop] = state.sol[0]
        if world > 1:
            sol_host[0] = comm.all_reduce_sum(sol_host[0], tag="bench")
        def e2e_step():
            st2 = P.PartitionedState([graph], part, solutions=sol_host)
            picks, applied = solve_step(st2, params, comm, sched, active)
            for v, a in zip(picks[0], applied[0]):
                if v >= 0 and a:
                    sol_host[0, v] = 1

        for _ in range(args.warmup):  # first states allocate their workspaces
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            e2e_step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        e2e_s = max_over_ranks(e0.elapsed_time(e1) / args.steps) / 1e3
        params_bytes = sum(a.nbytes for a in params.as_dict().values())
        e2e = {"value": e2e_s, "unit": "s",
               "h2d_bytes_per_step": int(graph.num_nodes + params_bytes + 64 * 4 + 8 * 8),
               "d2h_bytes_per_step": int(64 * 4 + 8 * 16 + 8 + 8 + 8),
               "path": "PartitionedState(graphs, part, solutions=host S) + solve_step"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cst, build = cpu_state(graph)
        est, detail = cpu_sample(cst, params.as_dict())
        detail["state_build_s"] = round(build, 2)
        cpu = {"value": est, "unit": "s", "cores": os.cpu_count(), "kind": "port",
               "sample": "oracle/port.py (reference numpy/scipy algorithm) on the same graph: "
                         f"1 timed embedding round x 5 + q + select + apply; {detail}"}

    train = None
    if not args.no_train:
        train = []
        ds2 = [P.generate_ba(10000, 4, 100 + i) for i in range(32)]
        leg2 = train_leg(P, comm, ds2, 32, 4, args.train_steps, args.warmup,
                         "MVC DQN training step, 32 x BA(10000,4,seed=100+i), K=64, T=5, tau=4 "
                         "(BASELINE configs[1])")
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            leg2["cpu_baseline"] = cpu_train_sample(ds2, 4, 32, 4)
        train.append(leg2)
        leg4 = train_leg(P, comm, [graph], 8, 4, max(2, args.train_steps // 2), 2,
                         f"MVC DQN training step, 8 tuples of BA({args.nodes},{args.m},0) "
                         "(node-level batch), K=64, T=5, tau=4 (BASELINE configs[3])")
        train.append(leg4)

    extra = None
    if not args.no_extra:
        extra = []
        g1 = P.generate_ba(1000, 4, 0)
        leg1 = infer_leg(P, comm, g1, 50, 5, "MVC inference step, BA(1000,4,seed=0), K=64, T=5 "
                                            "(BASELINE configs[0]; launch-bound)")
        t_solve, res = full_solve_leg(P, comm, g1)
        leg1["full_adaptive_solve_s"] = t_solve
        leg1["full_solve_cover"] = res.cover_size
        leg1["full_solve_evals"] = res.policy_evals
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            from oracle import port
            theta = P.PolicyParams.initialize(64, 5, seed=0).as_dict()
            t0 = time.perf_counter()
            (cover, evals, _, _), = port.solve([g1.edge_array], 1000, theta, 5)
            dt = time.perf_counter() - t0
            leg1["cpu_baseline"] = {"value": dt / evals, "unit": "s", "cores": os.cpu_count(),
                                    "kind": "port", "full_adaptive_solve_s": dt,
                                    "sample": f"oracle/port.py full adaptive solve ({evals} evals,"
                                              f" cover {len(cover)}) / evals"}
        extra.append(leg1)
        t0 = time.time()
        g5 = P.generate_rmat(args.rmat_scale, 16, 0)
        g5.csr_arrays()
        leg5 = infer_leg(P, comm, g5, 8, 2,
                         f"MVC inference step, R-MAT scale {args.rmat_scale} edge factor 16 "
                         "(a,b,c = .57,.19,.19, seed 0), K=64, T=5, first steps of the adaptive "
                         "episode (BASELINE configs[4])")
        leg5["graph_gen_s"] = round(time.time() - t0, 2)
        if args.full_episode and world == 1:
            t_solve, res = full_solve_leg(P, comm, g5)
            leg5["full_adaptive_solve_s"] = t_solve
            leg5["full_solve_cover"] = res.cover_size
            leg5["full_solve_evals"] = res.policy_evals
            leg5["full_solve_skipped"] = res.skipped
        extra.append(leg5)

    if rank == 0:
        line = {"metric": METRIC, "value": step_ms / 1e3, "unit": "s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms,
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic", "config": workload(args),
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clocks.summary(), "step_path": step_path,
                "train_steps": train,
                "other_inference": extra,
                "setup": {"graph_gen_s": round(t_gen, 2), "state_build_s": round(t_state, 3),
                          "alive_entries_at_start": alive_entries}}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
