"""Child process of tests/test_gpu_handle_abi.py: drives libs2v.so through
the handle-level C ABI (include/s2v.h, s2v_ctx / s2v_graph / s2v_state) with
plain ctypes + numpy -- torch is never imported -- against the reference's
golden fixtures.  Prints "OK <checks>" on success."""
import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import cref  # noqa: E402  (checker: the reference's BA generator restated)

GOLD = ROOT / "tests" / "golden"
lib = ctypes.CDLL(str(ROOT / "paper_2105_08764_b200" / "libs2v.so"))
P, I, I64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
lib.s2v_last_error.restype = ctypes.c_char_p
lib.s2v_graph_upload.argtypes = [P, I64, P, P, ctypes.POINTER(P)]
lib.s2v_state_create.argtypes = [P, P, I, P, ctypes.POINTER(P)]
lib.s2v_embed.argtypes = [P, P, I, P, I, I]
lib.s2v_global_sum.argtypes = [P, P, P]
lib.s2v_score_topk.argtypes = [P, P, I, P, P]
lib.s2v_apply.argtypes = [P, P, P, I, P, P]
lib.s2v_loss_grad.argtypes = [P, P, I, P, I, I, P, P, P, ctypes.POINTER(ctypes.c_double)]
lib.s2v_adam_update.argtypes = [P, I, P, P, P, P, I64, I, ctypes.c_double, ctypes.c_double,
                                ctypes.c_double, ctypes.c_double]
lib.s2v_copy_out.argtypes = [P, P, I, P]
for f in ("s2v_graph_destroy", "s2v_state_destroy", "s2v_ctx_destroy"):
    getattr(lib, f).argtypes = [P]
NAMES = [f"theta{i}" for i in range(1, 8)]


def ok(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: rc {rc}: {lib.s2v_last_error().decode()}")


def a(x):
    return x.ctypes.data_as(P)


def csr(n, edges):
    """Graph.csr_arrays(): symmetric CSR, ascending neighbour lists."""
    u = np.concatenate([edges[:, 0], edges[:, 1]])
    v = np.concatenate([edges[:, 1], edges[:, 0]])
    order = np.lexsort((v, u))
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(u, minlength=n), out=rp[1:])
    return rp, np.ascontiguousarray(v[order], dtype=np.int32)


def init_theta(K, L, seed):
    """PolicyParams.initialize(K, L, seed) (policy.py:79-102), packed."""
    rng = np.random.default_rng(seed)
    shapes = [(K, 1), (K, 1), (K, K), (K, K), (K, K), (K, K), (2 * K, 1)]
    th = [rng.uniform(-0.05, 0.05, size=s).astype(np.float32) for s in shapes]
    th[5] = np.abs(th[5])
    th[6][K:] = np.abs(th[6][K:])
    return np.concatenate([t.reshape(-1) for t in th])


def upload(ctx, n, m, seed):
    rp, cols = csr(n, cref.generate_ba_edges(n, m, seed))
    g = P()
    ok(lib.s2v_graph_upload(ctx, n, a(rp), a(cols), ctypes.byref(g)), "graph_upload")
    return g


def scale_error(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    return float(np.abs(x - y).max() / max(np.abs(x).max(), np.abs(y).max(), 1e-9))


def main():
    assert "torch" not in sys.modules
    ctx = P()
    ok(lib.s2v_ctx_create(0, 0, 1, None, ctypes.byref(ctx)), "ctx_create")
    checks = 0
    # -- forward: embeddings, g, scores bit for bit (fwd_ba1000_k64_l5) ---
    z = np.load(GOLD / "fwd_ba1000_k64_l5.npz")
    n, K, L = int(z["n"]), int(z["K"]), int(z["L"])
    g = upload(ctx, n, int(z["m"]), int(z["seed"]))
    st = P()
    graphs = (P * 1)(g)
    sol = np.ascontiguousarray(z["sol"][None], np.uint8)
    ok(lib.s2v_state_create(ctx, graphs, 1, a(sol), ctypes.byref(st)), "state_create")
    theta = init_theta(K, L, int(z["pseed"]))
    ok(lib.s2v_embed(ctx, st, 0, a(theta), K, L), "embed")
    h = np.empty((n, K), np.float32)
    ok(lib.s2v_copy_out(ctx, st, 0, a(h)), "copy_out h")
    assert np.array_equal(h, z["h"]), "embedding"
    gs = np.empty(K, np.float32)
    ok(lib.s2v_global_sum(ctx, st, a(gs)), "global_sum")
    assert np.array_equal(gs, z["g"]), "g"
    keys = np.empty((1, 8, 2), np.uint64)
    cnt = np.empty(1, np.int64)
    ok(lib.s2v_score_topk(ctx, st, 8, a(keys), a(cnt)), "score_topk")
    sc = np.empty(n, np.float32)
    ok(lib.s2v_copy_out(ctx, st, 5, a(sc)), "copy_out scores")
    cand = np.empty(n, np.uint8)
    ok(lib.s2v_copy_out(ctx, st, 2, a(cand)), "copy_out cand")
    assert np.array_equal(cand, z["cand"]), "cand"
    c = cand.astype(bool)
    assert np.array_equal(sc[c], z["scores"][c]), "scores"
    assert int(cnt[0]) == int(c.sum())
    top = np.flatnonzero(c)[np.argsort(-z["scores"][c], kind="stable")][:8]
    assert np.array_equal((~keys[0, :, 1]).astype(np.int64), top), "top-8 keys"
    checks += 6
    # apply: the reference's errors before anything is applied
    v = np.array([int(top[0])], np.int64)
    ok(lib.s2v_apply(ctx, st, a(v), 1, None, None), "apply")
    rc = lib.s2v_apply(ctx, st, a(v), 1, None, None)
    assert rc == 2 and b"already in the solution" in lib.s2v_last_error()
    ok(lib.s2v_copy_out(ctx, st, 1, a(cand)), "copy_out sol")
    assert cand[v[0]] == 1
    checks += 1
    lib.s2v_state_destroy(st)
    lib.s2v_graph_destroy(g)
    # -- full adaptive solve: cover, evaluations, skips (solve_ba1000_k64_l5) --
    z = np.load(GOLD / "solve_ba1000_k64_l5.npz")
    g = upload(ctx, 1000, 4, 0)
    st = P()
    ok(lib.s2v_state_create(ctx, (P * 1)(g), 1, None, ctypes.byref(st)), "state_create")
    theta = init_theta(int(z["K"]), int(z["L"]), int(z["pseed"]))
    cover, evals, skipped = [], 0, 0
    res = np.array([1], np.int64)
    while res[0] > 0:
        ok(lib.s2v_embed(ctx, st, 0, a(theta), int(z["K"]), int(z["L"])), "embed")
        ok(lib.s2v_score_topk(ctx, st, 8, a(keys), a(cnt)), "score_topk")
        c = int(cnt[0])
        d = next((dd for f, dd in ((0.5, 8), (0.25, 4), (0.125, 2)) if c > f * 1000), 1)
        d = min(d, c)  # SelectionSchedule.adaptive (inference.py:54-58)
        picks = np.ascontiguousarray((~keys[0, :d, 1]).astype(np.int64)[None])
        applied = np.zeros((1, d), np.uint8)
        ok(lib.s2v_apply(ctx, st, a(picks), d, a(applied), a(res)), "apply")
        cover += [int(v) for v, f in zip(picks[0], applied[0]) if f]
        skipped += int(d - applied.sum())
        evals += 1
    assert sorted(cover) == z["covers"].tolist(), "cover"
    assert evals == int(z["evals"][0]) and skipped == int(z["skipped"][0])
    checks += 2
    lib.s2v_state_destroy(st)
    lib.s2v_graph_destroy(g)
    # -- training step: grads, loss, Adam (train_ba1000_b4_k64_l5) ----------
    z = np.load(GOLD / "train_ba1000_b4_k64_l5.npz")
    n, B, K, L, tau = (int(z[k]) for k in ("n", "B", "K", "L", "tau"))
    gl = [upload(ctx, n, int(z["m"]), 100 + i) for i in range(B)]
    st = P()
    ok(lib.s2v_state_create(ctx, (P * B)(*gl), B, a(np.ascontiguousarray(z["snaps"], np.uint8)),
                            ctypes.byref(st)), "state_create")
    theta = np.concatenate([z[f"p0_{k}"].reshape(-1) for k in NAMES]).astype(np.float32)
    m = np.zeros_like(theta)
    v = np.zeros_like(theta)
    grads = np.empty_like(theta)
    loss = ctypes.c_double()
    acts = np.ascontiguousarray(z["actions"], np.int64)
    tg = np.ascontiguousarray(z["targets"], np.float32)
    for it in range(tau):
        ok(lib.s2v_loss_grad(ctx, st, 0, a(theta), K, L, a(acts), a(tg), a(grads),
                             ctypes.byref(loss)), "loss_grad")
        assert abs(loss.value - z["losses"][it]) <= 1e-4 * abs(z["losses"][it]), "loss"
        if it == 0:
            g0 = np.concatenate([z[f"g0_{k}"].reshape(-1) for k in NAMES])
            off = 0
            for k in NAMES:
                sz = z[f"g0_{k}"].size
                assert scale_error(grads[off:off + sz], g0[off:off + sz]) < 1e-4, k
                off += sz
        ok(lib.s2v_adam_update(ctx, 0, a(theta), a(grads), a(m), a(v), theta.size, it + 1,
                               1e-5, 0.9, 0.999, 1e-8), "adam")
    off = 0
    for k in NAMES:
        sz = z[f"p1_{k}"].size
        assert scale_error(theta[off:off + sz], z[f"p1_{k}"].reshape(-1)) < 1e-4, k
        assert scale_error(m[off:off + sz], z[f"m_{k}"].reshape(-1)) < 1e-4, k
        off += sz
    bad = grads.copy()
    bad[3] = np.nan
    before = theta.copy()
    rc = lib.s2v_adam_update(ctx, 0, a(theta), a(bad), a(m), a(v), theta.size, tau + 1, 1e-5,
                             0.9, 0.999, 1e-8)
    assert rc == 5 and np.array_equal(theta, before), "non-finite rejection"
    checks += 4
    lib.s2v_state_destroy(st)
    for x in gl:
        lib.s2v_graph_destroy(x)
    lib.s2v_ctx_destroy(ctx)
    assert "torch" not in sys.modules
    print("OK", checks)


if __name__ == "__main__":
    main()
