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
    ap.add_argument("--ref-steps", type=int, default=3,
                    help="reference arm: full steps actually run (>= 3, min reported)")
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


def reference_module():
    """The unmodified reference package graphrl, pip-installed from
    /root/reference into baseline/_ref (git-ignored; travels to the box).
    Returns (module, kind, description); falls back to oracle/port.py (the
    reference's numpy/scipy calls restated) when the install is absent."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "graphrl" / "__init__.py").exists():
        if str(ref) not in sys.path:
            sys.path.insert(0, str(ref))
        import graphrl
        return graphrl, "reference", ("graphrl 0.1.0 (pip install --target baseline/_ref "
                                      "/root/reference), its own public API")
    return None, "port", "oracle/port.py (reference numpy/scipy calls restated)"


def _libs2v_mapped() -> bool:
    """Whether this process mapped the product library (must be False for
    the reference arm)."""
    try:
        return "libs2v.so" in Path("/proc/self/maps").read_text()
    except Exception:
        return False


def host_info():
    """CPU model, logical cores and the BLAS pool the reference's numpy uses."""
    model = ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{k: d.get(k) for k in ("internal_api", "num_threads", "version", "architecture")}
                for d in threadpool_info() if d.get("user_api") == "blas"]
    except Exception:
        pass
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "blas": blas,
            "scipy_spmm_threads": 1}


def ref_inference_step(R, st, params, comm, sched, n):
    """One iteration of the reference's solve loop (inference.py:107-147)
    through its public API: embed_forward, q_forward, masked_scores, the
    select all-gather, d_for + select_top_d, group apply with the mid-group
    skip, residual_counts."""
    emb = R.embed_forward(st, params, comm)
    sc = R.q_forward(emb, st.cand, params, comm)
    gl = comm.all_gather(R.masked_scores(sc, st.cand), axis=-1, tag="select")
    cm = np.isfinite(gl[0])
    picks = R.select_top_d(gl[0], cm, sched.d_for(int(np.count_nonzero(cm)), n))
    for j, v in enumerate(picks):
        if j > 0 and not st.cand[0, v]:
            continue
        st.apply_action(v, slot=0)
    return st.residual_counts(comm)


def ref_graph(R, nodes, m):
    """The reference's Graph of generate_ba(nodes, m, 0), built from the
    edge array of the oracle's C restatement of generate_ba (pinned byte for
    byte against the reference; the reference's own Python loop takes
    216 s at 2M nodes).  The product library libs2v.so is never loaded."""
    from oracle import cref
    edges = cref.generate_ba_edges(nodes, m, 0)
    if R is None:
        return edges
    return R.Graph(nodes, edges)


def port_params(K, L, seed):
    """PolicyParams.initialize(K, L, seed) (policy.py:79-102) without the
    product package: one default_rng(seed) stream, theta1..theta7 in order,
    U(-0.05, 0.05) fp32, |theta6| and |theta7[K:]| ("positive")."""
    rng = np.random.default_rng(seed)
    shapes = [(K, 1), (K, 1), (K, K), (K, K), (K, K), (K, K), (2 * K, 1)]
    th = {f"theta{i + 1}": rng.uniform(-0.05, 0.05, size=sh).astype(np.float32)
          for i, sh in enumerate(shapes)}
    th["theta6"] = np.abs(th["theta6"])
    th["theta7"][K:] = np.abs(th["theta7"][K:])
    return th


def cpu_baseline_infer(graph):
    """cpu_baseline of the headline: ONE full inference step of the reference
    (from S = {}) on the same graph, this host's cores."""
    R, kind, desc = reference_module()
    if R is None:
        from oracle import port
        st = port.ResidualState([graph.edge_array], graph.num_nodes)
        t0 = time.perf_counter()
        port.inference_step(st, port_params(64, 5, 0), 5, np.array([True]))
        dt = time.perf_counter() - t0
    else:
        g = R.Graph(graph.num_nodes, graph.edge_array)
        params = R.PolicyParams.initialize(64, 5, seed=0)
        comm = R.WorkerGroup(1).comm(0)
        st = R.PartitionedState([g], R.partition_rows(graph.num_nodes, 1)[0])
        t0 = time.perf_counter()
        ref_inference_step(R, st, params, comm, R.SelectionSchedule.adaptive(), graph.num_nodes)
        dt = time.perf_counter() - t0
    return {"value": dt, "unit": "s", "cores": os.cpu_count(), "kind": kind,
            "sample": f"{desc}: one full inference step (5 rounds + q + select + apply) from "
                      f"S = {{}} on the same graph", "host": host_info()}


def run_reference(args):
    """--impl reference: the reference's own CPU inference step, timed on
    this host, rank 0 only.  Each step is one full policy evaluation +
    selection + apply of the episode from S = {}; min over the steps that
    actually ran (at least 3)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    R, kind, desc = reference_module()
    t0 = time.perf_counter()
    g = ref_graph(R, args.nodes, args.m)
    t_graph = time.perf_counter() - t0
    nsteps = max(3, args.ref_steps)
    if R is not None:
        params = R.PolicyParams.initialize(64, 5, seed=0)
        comm = R.WorkerGroup(1).comm(0)
        t0 = time.perf_counter()
        st = R.PartitionedState([g], R.partition_rows(args.nodes, 1)[0])
        t_build = time.perf_counter() - t0
        sched = R.SelectionSchedule.adaptive()
        times = []
        for _ in range(nsteps):
            t0 = time.perf_counter()
            ref_inference_step(R, st, params, comm, sched, args.nodes)
            times.append(time.perf_counter() - t0)
    else:  # port fallback: the same loop body, restated (oracle/port.py)
        from oracle import port
        theta = port_params(64, 5, 0)
        t0 = time.perf_counter()
        st = port.ResidualState([g], args.nodes)
        t_build = time.perf_counter() - t0
        times = []
        for _ in range(nsteps):
            t0 = time.perf_counter()
            port.inference_step(st, theta, 5, np.array([True]))
            times.append(time.perf_counter() - t0)
    value = float(min(times))
    info = host_info()
    sample = (f"{desc}: {nsteps} full inference steps (embed_forward 5 rounds + q_forward + "
              f"select all-gather + top-d + group apply + residual_counts) of the adaptive "
              f"episode from S = {{}}, min over steps; step times "
              f"{[round(t, 2) for t in times]} s; graph {t_graph:.1f}s and PartitionedState "
              f"build {t_build:.1f}s excluded")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "s",
            "n_gpus": args.gpus, "steps": nsteps, "warmup": 0,
            "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": workload(args),
            "cpu_baseline": {"value": value, "unit": "s", "cores": os.cpu_count(), "kind": kind,
                             "sample": sample, "host": info},
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "step_times_s": times, "mean_step_s": float(np.mean(times)),
            "product_library_mapped": _libs2v_mapped(),
            "setup": {"graph_s": round(t_graph, 2), "state_build_s": round(t_build, 2)}}
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
    value = e0.elapsed_time(e1) / steps / 1e3
    # roofline of the backward kernels: per-launch CUDA events over one more
    # step (policy.BWD_TIMER), algorithmic bytes per launch from the batch
    from paper_2105_08764_b200 import policy
    policy.BWD_TIMER = []
    P.train_step(buf, dataset, params, adam, cfg, rng, comm, part)
    torch.cuda.synchronize()
    timer, policy.BWD_TIMER = policy.BWD_TIMER, None
    return {"workload": name, "value": value, "unit": "s",
            "B": B, "tau": tau, "steps": steps, "warmup": warmup,
            "last_losses": [float(x) for x in losses],
            "path": "train_step(buffer, dataset, params, adam, cfg, rng, comm, part)",
            "roofline": train_roofline(buf, dataset, B, part, timer)}


def train_roofline(buf, dataset, B, part, timer):
    """HBM roofline of the two backward kernels of loss_and_gradients at this
    batch: spmm_t (s2v_gather, the dominant training kernel) and the
    tcgen05 layer backward.  Bytes per launch (fp32, K = 64, rows = B x
    local rows): gather 8(rows+1) + 4 nnz + 256 alive entries + 256 rows;
    layer backward 256 rows x (grad_h + h_l [+ dzsum in] + dzsum out [+ m]
    [+ dm out])."""
    rows = B * part.num_rows
    nnz = alive = 0
    for i in range(min(B, len(buf))):
        t = buf[i]
        g = dataset[t.graph_index]
        sol = np.unpackbits(np.frombuffer(t.solution_snapshot, np.uint8))[
            :g.num_nodes].astype(bool)
        e = g.edge_array
        nnz += 2 * len(e)
        alive += 2 * int(np.count_nonzero(~sol[e[:, 0]] & ~sol[e[:, 1]]))
    peak, peak_src = peaks()
    out = {"peak": peak, "peak_source": peak_src, "unit": "GB/s", "bound": "hbm"}
    for tag, model in (("gather", lambda f: 8 * (rows + 1) + 4 * nnz + 256 * alive + 256 * rows),
                       ("layer_backward",
                        lambda f: 256 * rows * (2 + (0 if f[0] else 1) + 1 + int(f[1]) +
                                                int(f[2])))):
        ev = [(t, a, b) for t, a, b in timer if t[0] == tag]
        if not ev:
            continue
        ms = [a.elapsed_time(b) for _, a, b in ev]
        byts = [model(t[1:]) for t, _, _ in ev]
        achieved = sum(byts) / (sum(ms) * 1e-3) / 1e9
        out[tag] = {"achieved": round(achieved, 1), "frac": round(achieved / peak, 4),
                    "avg_launch_ms": round(float(np.mean(ms)), 4), "launches": len(ev),
                    "algorithmic_bytes_per_launch": int(np.mean(byts))}
    out["kernels"] = {"gather": "gather64_tiles_kernel (spmm_t, the dominant training kernel)",
                      "layer_backward": "layer_backward64_tc_kernel (tcgen05 split-TF32 dm and "
                                        "dtheta4, fused dz / dzsum)"}
    if "gather" in out:
        out.update({"achieved": out["gather"]["achieved"], "frac": out["gather"]["frac"]})
    return out


def cpu_baseline_train(P, dataset, B, tau):
    """BASELINE configs[1] on the CPU: ONE full train_step of the reference
    (tuples_to_graphs + batch_targets + tau x (loss_and_gradients +
    adam_step)) on the same B tuples, this host's cores."""
    R, kind, desc = reference_module()
    buf = _train_buffer(P, dataset, B)
    if R is None:
        return None
    graphs = [R.Graph(g.num_nodes, g.edge_array) for g in dataset]
    rbuf = R.ReplayBuffer(max(B, 1))
    for i in range(len(buf)):
        t = buf[i]
        rbuf.add(R.ExperienceTuple(t.graph_index, t.solution_snapshot, t.action, 0.0))
    params = R.PolicyParams.initialize(64, 5, seed=0)
    adam = R.AdamState.create(params, lr=1e-5)
    cfg = R.TrainConfig(embed_dim=64, num_layers=5, batch_size=B, tau=tau)
    comm = R.WorkerGroup(1).comm(0)
    part = R.partition_rows(dataset[0].num_nodes, 1)[0]
    t0 = time.perf_counter()
    R.train_step(rbuf, graphs, params, adam, cfg, np.random.default_rng(7), comm, part)
    dt = time.perf_counter() - t0
    return {"value": dt, "unit": "s", "cores": os.cpu_count(), "kind": kind,
            "sample": f"{desc}: one full train_step (B={B}, tau={tau}) on the same tuples"}


def cpu_baseline_cfg4(graph, B, tau, L=5, K=64):
    """BASELINE configs[3] on the CPU, bounded sample (the full step is
    ~10^3-10^4 s): on one tuple of the same graph, time the reference's
    PartitionedState build, one embedding round (policy.py:163-174:
    state.spmm + theta4 matmul + relu) and one backward layer
    (policy.py:290-304: the three einsums, two matmuls, state.spmm_t), then
    scale to train_step's B x (state build x 2 + L forward rounds for the
    targets) + tau x B x L x (forward round + backward layer)."""
    R, kind, desc = reference_module()
    if R is None:
        return None
    n = graph.num_nodes
    g = R.Graph(n, graph.edge_array)
    t0 = time.perf_counter()
    st = R.PartitionedState([g], R.partition_rows(n, 1)[0])
    t_state = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    th = {k: v for k, v in R.PolicyParams.initialize(K, L, seed=0).as_dict().items()}
    h = np.abs(rng.normal(size=(1, K, n))).astype(np.float32)
    e12 = rng.normal(size=(1, K, n)).astype(np.float32)
    t0 = time.perf_counter()
    m = np.ascontiguousarray(st.spmm(h))
    z = e12 + np.matmul(th["theta4"], m)
    h2 = np.maximum(z, 0)
    t_fwd = time.perf_counter() - t0
    w = np.abs(rng.normal(size=(1, K, n))).astype(np.float32)
    sol = np.zeros((1, n), np.float32)
    t0 = time.perf_counter()
    dz = h2 * (z > 0)
    np.einsum("bkv,bv->k", dz, sol)
    np.einsum("bkv,bjv->kj", dz, w)
    np.matmul(th["theta3"].T, dz)
    np.einsum("bkv,bjv->kj", dz, m)
    st.spmm_t(np.matmul(th["theta4"].T, dz))
    t_bwd = time.perf_counter() - t0
    est = B * (2 * t_state + L * t_fwd) + tau * B * L * (t_fwd + t_bwd)
    return {"value": est, "unit": "s", "cores": os.cpu_count(), "kind": kind,
            "sample": f"{desc} building blocks on 1 tuple of the same graph: PartitionedState "
                      f"{t_state:.2f}s, forward round {t_fwd:.2f}s, backward layer {t_bwd:.2f}s;"
                      f" scaled as B*(2*state + L*fwd) + tau*B*L*(fwd + bwd), B={B}, "
                      f"tau={tau}, L={L} (an estimate: the measured full reference step at "
                      "B=2, tau=1 is 531 s, SURVEY.md section 6)"}


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
        tr = json.loads((ROOT / "profiles" / "r2s3_round64_traffic.json").read_text())
        if args.nodes == 2_000_000 and args.m == 16 and world == 1:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "traffic_source": "profiles/r2s3_round64_traffic.json (ncu dram__bytes_read+write)",
                "kernel": "round64_kernel (fused gather-SpMM + theta4 FMA chain + e12 + relu), "
                          "rounds 3..5 (round 2 gathers the per-degree h1 table, round 1 is "
                          "skipped)",
                "round_ms": round(round_ms, 4), "algorithmic_bytes_per_launch": algo_bytes,
                "peak_source": peak_src,
                "bytes_model": "8(rows+1) row_ptr + 4 nnz cols + 256 alive gathers + 256 rows h_out"
                               " + 4 rows rdeg + rows sol"}
    if world > 1:
        # NVLink roofline of the fused halo exchange: every round pushes this
        # rank's new rows into every peer, so each GPU receives the other
        # ranks' rows, 4 K (N - N_loc) bytes per round,
        # during the round kernel (round_ms includes the push)
        recv = 4 * 64 * (graph.num_nodes - rows)
        nv_peak = 770.0  # GB/s per direction, measured peer copy (B200_PROFILING.md)
        nv = recv / (round_ms * 1e-3) / 1e9
        roofline["nvlink"] = {
            "bytes_received_per_round": recv, "achieved": round(nv, 1), "peak": nv_peak,
            "unit": "GB/s", "frac": round(nv / nv_peak, 4),
            "peak_source": "measured peer copy per direction (B200_PROFILING.md)",
            "transport": type(comm.device_comm()).__name__,
            "same_device": bool(args.same_device),
            "note": ("ranks share one GPU: no NVLink traversed, the fraction is not an NVLink "
                     "measurement") if args.same_device else "fused push over NVLink P2P"}

    # end to end through the public API: host solution vector -> state -> step
    e2e = None
    if not args.no_e2e:
        sol_host = np.zeros((1, graph.num_nodes), dtype=np.uint8)
        sol_host[0, part.row_start:part.row_stop] = state.sol[0]
        if world > 1:
            sol_host[0] = comm.all_reduce_sum(sol_host[0], tag="bench")
        held = []

        def e2e_step():
            # the caller drops the previous step's state before building the
            # next (its device buffers go back to the caching allocator now,
            # not whenever Python's cycle collector runs)
            while held:
                held.pop().release()
            st2 = P.PartitionedState([graph], part, solutions=sol_host)
            held.append(st2)
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
        cpu = cpu_baseline_infer(graph)

    train = None
    if not args.no_train:
        train = []
        ds2 = [P.generate_ba(10000, 4, 100 + i) for i in range(32)]
        leg2 = train_leg(P, comm, ds2, 32, 4, args.train_steps, args.warmup,
                         "MVC DQN training step, 32 x BA(10000,4,seed=100+i), K=64, T=5, tau=4 "
                         "(BASELINE configs[1])")
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            leg2["cpu_baseline"] = cpu_baseline_train(P, ds2, 32, 4)
        train.append(leg2)
        leg4 = train_leg(P, comm, [graph], 8, 4, max(2, args.train_steps // 2), 2,
                         f"MVC DQN training step, 8 tuples of BA({args.nodes},{args.m},0) "
                         "(node-level batch), K=64, T=5, tau=4 (BASELINE configs[3])")
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            leg4["cpu_baseline"] = cpu_baseline_cfg4(graph, 8, 4)
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
            R, kind, desc = reference_module()
            if R is not None:
                rg = R.Graph(1000, g1.edge_array)
                rp = R.PolicyParams.initialize(64, 5, seed=0)
                t0 = time.perf_counter()
                (rr,) = R.run_workers(1, lambda c: R.solve([rg], rp, c))[0]
                dt = time.perf_counter() - t0
                cover_n, evals = rr.cover_size, rr.policy_evals
            else:
                from oracle import port
                t0 = time.perf_counter()
                (cover, evals, _, _), = port.solve([g1.edge_array], 1000, port_params(64, 5, 0),
                                                   5)
                dt = time.perf_counter() - t0
                cover_n = len(cover)
            leg1["cpu_baseline"] = {"value": dt / evals, "unit": "s", "cores": os.cpu_count(),
                                    "kind": kind, "full_adaptive_solve_s": dt,
                                    "sample": f"{desc}: full adaptive solve ({evals} evals, "
                                              f"cover {cover_n}) / evals"}
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
