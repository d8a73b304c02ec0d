"""Child process of tests/test_gpu_handle_abi.py: drives libs2v.so through
the handle-level C ABI (include/s2v.h, s2v_ctx / s2v_graph / s2v_state) with
plain ctypes + numpy -- torch is never imported -- against the reference's
golden fixtures, single-rank and node-sharded (P = 2, 3 thread ranks of
one in-process group sharing the GPU).  Prints "OK <checks>" on success."""
import ctypes
import sys
import threading
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
lib.s2v_group_create.argtypes = [I, ctypes.POINTER(P)]
lib.s2v_ctx_create_in_group.argtypes = [I, I, P, ctypes.POINTER(P)]
for f in ("s2v_graph_destroy", "s2v_state_destroy", "s2v_ctx_destroy", "s2v_group_destroy"):
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


def part(n, world, rank):
    """partition_rows(n, world)[rank] (state.py:36-53): (start, rows)."""
    base, extra = divmod(n, world)
    return rank * base + min(rank, extra), base + (1 if rank < extra else 0)


def forward_checks(ctx, rank, world):
    """fwd_ba1000_k64_l5: embeddings, g, scores bit for bit; the apply errors."""
    z = np.load(GOLD / "fwd_ba1000_k64_l5.npz")
    n, K, L = int(z["n"]), int(z["K"]), int(z["L"])
    r0, rows = part(n, world, rank)
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
    sc = np.empty(rows, np.float32)
    ok(lib.s2v_copy_out(ctx, st, 5, a(sc)), "copy_out scores")
    cand = np.empty(rows, np.uint8)
    ok(lib.s2v_copy_out(ctx, st, 2, a(cand)), "copy_out cand")
    assert np.array_equal(cand, z["cand"][r0:r0 + rows]), "cand"
    c = cand.astype(bool)
    assert np.array_equal(sc[c], z["scores"][r0:r0 + rows][c]), "scores"
    call = z["cand"].astype(bool)
    assert int(cnt[0]) == int(call.sum())
    top = np.flatnonzero(call)[np.argsort(-z["scores"][call], kind="stable")][:8]
    assert np.array_equal((~keys[0, :, 1]).astype(np.int64), top), "top-8 keys"
    # apply: the reference's errors before anything is applied (at P > 1 the
    # owner's verdict reaches every rank)
    v = np.array([int(top[0])], np.int64)
    ok(lib.s2v_apply(ctx, st, a(v), 1, None, None), "apply")
    rc = lib.s2v_apply(ctx, st, a(v), 1, None, None)
    assert rc == 2 and b"already in the solution" in lib.s2v_last_error()
    sol_l = np.empty(rows, np.uint8)
    ok(lib.s2v_copy_out(ctx, st, 1, a(sol_l)), "copy_out sol")
    if r0 <= v[0] < r0 + rows:
        assert sol_l[v[0] - r0] == 1
    lib.s2v_state_destroy(st)
    lib.s2v_graph_destroy(g)
    return 7


def solve_checks(ctx):
    """solve_ba1000_k64_l5: the whole adaptive trajectory."""
    z = np.load(GOLD / "solve_ba1000_k64_l5.npz")
    g = upload(ctx, 1000, 4, 0)
    st = P()
    ok(lib.s2v_state_create(ctx, (P * 1)(g), 1, None, ctypes.byref(st)), "state_create")
    theta = init_theta(int(z["K"]), int(z["L"]), int(z["pseed"]))
    keys = np.empty((1, 8, 2), np.uint64)
    cnt = np.empty(1, np.int64)
    cover, evals, skipped = [], 0, 0
    while True:
        ok(lib.s2v_embed(ctx, st, 0, a(theta), int(z["K"]), int(z["L"])), "embed")
        ok(lib.s2v_score_topk(ctx, st, 8, a(keys), a(cnt)), "score_topk")
        c = int(cnt[0])
        if c == 0:
            break
        d = next((dd for f, dd in ((0.5, 8), (0.25, 4), (0.125, 2)) if c > f * 1000), 1)
        d = min(d, c)  # SelectionSchedule.adaptive (inference.py:54-58)
        picks = np.ascontiguousarray((~keys[0, :d, 1]).astype(np.int64)[None])
        applied = np.zeros((1, d), np.uint8)
        ok(lib.s2v_apply(ctx, st, a(picks), d, a(applied), None), "apply")
        cover += [int(v) for v, f in zip(picks[0], applied[0]) if f]
        skipped += int(d - applied.sum())
        evals += 1
    assert sorted(cover) == z["covers"].tolist(), "cover"
    assert evals == int(z["evals"][0]) and skipped == int(z["skipped"][0])
    lib.s2v_state_destroy(st)
    lib.s2v_graph_destroy(g)
    return 2


def train_checks(ctx):
    """train_ba1000_b4_k64_l5: loss, grads, Adam over tau steps.  Returns
    the first step's gradients (replicas must agree at P > 1)."""
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
    first = None
    for it in range(tau):
        ok(lib.s2v_loss_grad(ctx, st, 0, a(theta), K, L, a(acts), a(tg), a(grads),
                             ctypes.byref(loss)), "loss_grad")
        assert abs(loss.value - z["losses"][it]) <= 1e-4 * abs(z["losses"][it]), "loss"
        if it == 0:
            first = (loss.value, grads.copy())
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
    lib.s2v_state_destroy(st)
    for x in gl:
        lib.s2v_graph_destroy(x)
    return 4, first


def run_ranks(world, fn):
    """fn(ctx, rank) on `world` thread ranks of one in-process group (all on
    GPU 0); returns the per-rank results, raising the first failure."""
    grp = P()
    ok(lib.s2v_group_create(world, ctypes.byref(grp)), "group_create")
    out, errs = [None] * world, []

    def body(rank):
        ctx = P()
        try:
            ok(lib.s2v_ctx_create_in_group(0, rank, grp, ctypes.byref(ctx)), "ctx_create_in_group")
            out[rank] = fn(ctx, rank)
        except BaseException as e:  # noqa: BLE001 (reported by the caller)
            errs.append(f"rank {rank}: {e!r}")
        finally:
            lib.s2v_ctx_destroy(ctx)
    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    lib.s2v_group_destroy(grp)
    if errs:
        raise AssertionError("; ".join(errs))
    return out


def main():
    assert "torch" not in sys.modules
    ctx = P()
    ok(lib.s2v_ctx_create(0, 0, 1, None, ctypes.byref(ctx)), "ctx_create")
    checks = forward_checks(ctx, 0, 1) + solve_checks(ctx)
    c, (loss1, grads1) = train_checks(ctx)
    checks += c
    lib.s2v_ctx_destroy(ctx)
    # node-sharded: the same goldens at P = 2, 3 thread ranks, every rank
    # returning the same keys, trajectory, loss and gradients
    for world in (2, 3):
        checks += sum(run_ranks(world, lambda c, r: forward_checks(c, r, world)))
        checks += sum(run_ranks(world, lambda c, r: solve_checks(c)))
        res = run_ranks(world, lambda c, r: train_checks(c))
        for c, (loss, grads) in res:
            checks += c
            assert loss == res[0][1][0] and np.array_equal(grads, res[0][1][1]), "replicas"
            assert abs(loss - loss1) <= 1e-6 * abs(loss1)
            assert scale_error(grads, grads1) < 1e-5, "P-invariant gradients"
    assert "torch" not in sys.modules
    print("OK", checks)


if __name__ == "__main__":
    main()
