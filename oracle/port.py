"""Single-rank numpy/scipy restatement of the reference's hot path.

TEST INFRASTRUCTURE ONLY -- imported by tests/ (as the checker for the
training path and the selection loop) and by bench.py's cpu_baseline /
--impl reference legs (as the reference's CPU implementation, timed on the
host).  The product package never imports it.

It follows the reference algorithm call for call, with the same numpy/scipy
operations in the same layouts, so that its fp32 results are those of the
reference at P=1 (pinned by tests/test_oracle.py against golden vectors the
reference itself produced, tests/golden/).  Paths are relative to
/root/reference:

  ResidualState      pkg/src/graphrl/state.py:65-220   (P = 1: all rows local)
  embed / q / mask   pkg/src/graphrl/policy.py:144-224
  loss_and_grads     pkg/src/graphrl/policy.py:232-315
  adam               pkg/src/graphrl/policy.py:339-359
  select_top_d       pkg/src/graphrl/inference.py:61-73
  solve_batch        pkg/src/graphrl/inference.py:90-152
  batch_targets      pkg/src/graphrl/agent.py:205-232
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

NAMES = ("theta1", "theta2", "theta3", "theta4", "theta5", "theta6", "theta7")


def _relu(x):
    return np.maximum(x, 0)


class ResidualState:
    """B graphs (same N) stacked block-diagonally; removed entries are zero
    values of one fixed CSR (state.py:89-111)."""

    def __init__(self, edge_arrays, n, solutions=None, dtype=np.float32):
        self.n, self.batch, self.dtype = n, len(edge_arrays), np.dtype(dtype)
        if solutions is None:
            solutions = np.zeros((self.batch, n), dtype=np.uint8)
        solutions = np.asarray(solutions, dtype=np.uint8)
        rows, cols, vals = [], [], []
        for b, e in enumerate(edge_arrays):
            e = np.asarray(e, dtype=np.int64).reshape(-1, 2)
            r = np.concatenate([e[:, 0], e[:, 1]])
            c = np.concatenate([e[:, 1], e[:, 0]])
            alive = (solutions[b, r] == 0) & (solutions[b, c] == 0)
            rows.append(r + b * n)
            cols.append(c + b * n)
            vals.append(alive.astype(self.dtype))
        self.mat = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows),
                                                         np.concatenate(cols))),
                                 shape=(self.batch * n, self.batch * n))
        idx = self.mat.indices
        self.col_order = np.argsort(idx, kind="stable")
        self.col_ptr = np.zeros(self.mat.shape[1] + 1, dtype=np.int64)
        np.cumsum(np.bincount(idx, minlength=self.mat.shape[1]), out=self.col_ptr[1:])
        self.sol = solutions.copy()
        self.cand = ((self.degrees() > 0) & (self.sol == 0)).astype(np.uint8)
        self.residual = np.array([np.count_nonzero(
            self.mat.data[self.mat.indptr[b * n]:self.mat.indptr[(b + 1) * n]])
            for b in range(self.batch)], dtype=np.int64)

    def degrees(self):
        return np.asarray(self.mat.sum(axis=1)).ravel().reshape(self.batch, self.n)

    def spmm(self, h):
        b, k, n = h.shape
        out = h.transpose(1, 0, 2).reshape(k, b * n) @ self.mat
        return out.reshape(k, b, n).transpose(1, 0, 2)

    def spmm_t(self, m):
        b, k, n = m.shape
        out = m.transpose(1, 0, 2).reshape(k, b * n) @ self.mat.T
        return out.reshape(k, b, n).transpose(1, 0, 2)

    def apply(self, v, slot=0):
        n = self.n
        data, indptr = self.mat.data, self.mat.indptr
        if self.sol[slot, v]:
            raise ValueError(f"node {v} is already in the solution")
        if not self.cand[slot, v]:
            raise ValueError(f"node {v} is not a candidate")
        r = slot * n + v
        removed = int(np.count_nonzero(data[indptr[r]:indptr[r + 1]]))
        data[indptr[r]:indptr[r + 1]] = 0
        self.sol[slot, v] = 1
        self.cand[slot, v] = 0
        c = slot * n + v
        ent = self.col_order[self.col_ptr[c]:self.col_ptr[c + 1]]
        removed += int(np.count_nonzero(data[ent]))
        data[ent] = 0
        self.residual[slot] -= removed
        sums = np.asarray(self.mat[slot * n:(slot + 1) * n].sum(axis=1)).ravel()
        self.cand[slot] = ((sums > 0) & (self.sol[slot] == 0)).astype(np.uint8)


def embed(state: ResidualState, theta: dict, num_layers: int, tape: bool = False):
    dt = theta["theta1"].dtype
    sol = state.sol.astype(dt)
    deg = state.degrees().astype(dt)
    w = _relu(theta["theta2"][:, 0][None, :, None] * deg[:, None, :])
    e1 = theta["theta1"][:, 0][None, :, None] * sol[:, None, :]
    e2 = np.matmul(theta["theta3"], w)
    h = np.zeros((state.batch, theta["theta1"].shape[0], state.n), dtype=dt)
    masks, ms = [], []
    for _ in range(num_layers):
        # the reference's all-reduce returns a C-contiguous copy (collective.py:113)
        m = np.ascontiguousarray(state.spmm(h))
        z = e1 + e2 + np.matmul(theta["theta4"], m)
        if tape:
            masks.append(z > 0)
            ms.append(m)
        h = _relu(z)
    if tape:
        return h, {"sol": sol, "deg": deg, "w": w, "masks": masks, "ms": ms}
    return h


def scores(h, cand, theta, tape: bool = False):
    dt = theta["theta1"].dtype
    c = cand.astype(dt)
    g = h.sum(axis=2)
    u1 = g @ theta["theta5"].T
    u2 = np.matmul(theta["theta6"], h * c[:, None, :])
    pre = np.concatenate([np.broadcast_to(u1[:, :, None], u2.shape), u2], axis=1)
    r = _relu(pre)
    s = np.einsum("bjv,j->bv", r, theta["theta7"][:, 0])
    if tape:
        return s, {"g": g, "pre": pre, "r": r}
    return s


def masked(s, cand):
    return np.where(cand.astype(bool), s, np.array(-np.inf, dtype=s.dtype))


def select_top_d(s, cand, d):
    idx = np.flatnonzero(np.asarray(cand, dtype=bool))
    if idx.size == 0:
        raise ValueError("empty candidate set")
    order = np.argsort(-np.asarray(s)[idx], kind="stable")
    return [int(idx[i]) for i in order[:min(d, idx.size)]]


def d_for(num_cand, n, thresholds=((0.5, 8), (0.25, 4), (0.125, 2)), fallback=1):
    for frac, d in thresholds:
        if num_cand > frac * n:
            return d
    return fallback


def inference_step(state: ResidualState, theta, num_layers, active, schedule=None):
    """One iteration of _solve_batch's loop (inference.py:107-147) at P=1."""
    schedule = schedule or {}
    h = embed(state, theta, num_layers)
    gl = masked(scores(h, state.cand, theta), state.cand)
    picks = []
    for b in range(state.batch):
        if not active[b]:
            picks.append([])
            continue
        cm = np.isfinite(gl[b])
        d = d_for(int(np.count_nonzero(cm)), state.n, **schedule)
        picks.append(select_top_d(gl[b], cm, d))
    applied = [[] for _ in range(state.batch)]
    skipped = np.zeros(state.batch, dtype=np.int64)
    for j in range(max((len(p) for p in picks), default=0)):
        for b in range(state.batch):
            if j >= len(picks[b]):
                continue
            v = picks[b][j]
            if j > 0 and not state.cand[b, v]:
                skipped[b] += 1
                continue
            state.apply(v, b)
            applied[b].append(v)
    return picks, applied, skipped


def solve(edge_arrays, n, theta, num_layers, schedule=None):
    """Full episode; returns per graph (cover, evals, skipped, picks per eval)."""
    st = ResidualState(edge_arrays, n, dtype=theta["theta1"].dtype)
    active = st.residual > 0
    covers = [[] for _ in range(st.batch)]
    evals = np.zeros(st.batch, dtype=np.int64)
    skipped = np.zeros(st.batch, dtype=np.int64)
    trace = [[] for _ in range(st.batch)]
    while np.any(active):
        picks, applied, sk = inference_step(st, theta, num_layers, active, schedule)
        for b in range(st.batch):
            if active[b]:
                evals[b] += 1
                trace[b].append(picks[b])
                covers[b].extend(applied[b])
        skipped += sk
        active = st.residual > 0
    return [(sorted(covers[b]), int(evals[b]), int(skipped[b]), trace[b])
            for b in range(st.batch)]


def loss_and_grads(state: ResidualState, actions, targets, theta, num_layers):
    """loss_and_gradients at P=1 (policy.py:232-315)."""
    b, n = state.batch, state.n
    k = theta["theta1"].shape[0]
    dt = theta["theta1"].dtype
    actions = np.asarray(actions, dtype=np.int64)
    targets = np.asarray(targets, dtype=dt)
    onehot = np.zeros((b, n), dtype=np.uint8)
    onehot[np.arange(b), actions] = 1
    h, et = embed(state, theta, num_layers, tape=True)
    s, qt = scores(h, onehot, theta, tape=True)
    grads = {name: np.zeros_like(theta[name]) for name in NAMES}
    dh = np.zeros_like(h)
    dg = np.zeros((b, k), dtype=dt)
    sq = 0.0
    for i in range(b):
        a = actions[i]
        err = s[i, a] - targets[i]
        sq += float(err) ** 2
        delta = 2.0 * err / b
        dpre = delta * theta["theta7"][:, 0] * (qt["pre"][i, :, a] > 0)
        grads["theta7"] += (delta * qt["r"][i, :, a])[:, None]
        grads["theta5"] += np.outer(dpre[:k], qt["g"][i])
        grads["theta6"] += np.outer(dpre[k:], h[i, :, a])
        dg[i] = theta["theta5"].T @ dpre[:k]
        dh[i, :, a] += theta["theta6"].T @ dpre[k:]
    dh += dg[:, :, None]
    dw = np.zeros_like(et["w"])
    gh = dh
    for layer in range(num_layers - 1, -1, -1):
        dz = gh * et["masks"][layer]
        grads["theta1"][:, 0] += np.einsum("bkv,bv->k", dz, et["sol"])
        grads["theta3"] += np.einsum("bkv,bjv->kj", dz, et["w"])
        dw += np.matmul(theta["theta3"].T, dz)
        grads["theta4"] += np.einsum("bkv,bjv->kj", dz, et["ms"][layer])
        if layer == 0:
            break
        gh = state.spmm_t(np.matmul(theta["theta4"].T, dz))
    grads["theta2"][:, 0] = np.einsum("bkv,bv->k", dw * (et["w"] > 0), et["deg"])
    return sq / b, grads


def adam(theta, grads, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """In-place bias-corrected Adam (policy.py:339-359); returns step + 1."""
    step += 1
    b1c = 1.0 - beta1 ** step
    b2c = 1.0 - beta2 ** step
    for name in NAMES:
        g = grads[name]
        m[name] = beta1 * m[name] + (1 - beta1) * g
        v[name] = beta2 * v[name] + (1 - beta2) * g * g
        upd = lr * (m[name] / b1c) / (np.sqrt(v[name] / b2c) + eps)
        theta[name] -= upd.astype(theta[name].dtype)
    return step


def batch_targets(edge_arrays, n, snapshots, actions, theta, num_layers, gamma):
    """Bellman targets at sampling time (agent.py:205-232), MVC reward -1."""
    dt = theta["theta1"].dtype
    nxt = np.asarray(snapshots, dtype=np.uint8).copy()
    nxt[np.arange(len(actions)), actions] = 1
    st = ResidualState(edge_arrays, n, solutions=nxt, dtype=dt)
    counts = st.residual.copy()
    h = embed(st, theta, num_layers)
    gl = masked(scores(h, st.cand, theta), st.cand)
    rewards = np.full(len(actions), -1.0, dtype=dt)
    return np.where(counts == 0, rewards, rewards + gamma * gl.max(axis=1))
