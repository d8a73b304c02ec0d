"""ctypes binding of the C++ op-order oracle (oracle/libs2v_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline leg of bench.py as the checker.  Never imported by the product
package.  See s2v_oracle.cpp for the reference file:line each routine follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "libs2v_oracle.so"

_lib = None


def build() -> Path:
    """Compile the oracle with its Makefile (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists() or (
                LIB_PATH.stat().st_mtime < (HERE / "s2v_oracle.cpp").stat().st_mtime):
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int
        L.s2vo_degrees.argtypes = [i64, P, P, P, P]
        for suf in ("f32", "f64"):
            getattr(L, f"s2vo_embed_{suf}").argtypes = [i64, P, P, P, P, P, P, P, i32, i32, P]
            getattr(L, f"s2vo_embed_{suf}").restype = i32
            getattr(L, f"s2vo_colsum_{suf}").argtypes = [i64, i32, P, P]
            getattr(L, f"s2vo_scores_{suf}").argtypes = [i64, i32, P, P, P, P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _suffix(dtype) -> str:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise ValueError(f"unsupported dtype {dt}")


def csr_of(graph_or_edges, n: int | None = None):
    """Symmetric CSR (int64 row_ptr, int32 sorted cols) of an edge array."""
    if hasattr(graph_or_edges, "edge_array"):
        n = graph_or_edges.num_nodes
        edges = np.asarray(graph_or_edges.edge_array, dtype=np.int64)
    else:
        edges = np.asarray(graph_or_edges, dtype=np.int64).reshape(-1, 2)
    rows = np.concatenate([edges[:, 0], edges[:, 1]])
    cols = np.concatenate([edges[:, 1], edges[:, 0]])
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    return row_ptr, cols.astype(np.int32)


def degrees(row_ptr, cols, sol) -> np.ndarray:
    n = len(row_ptr) - 1
    out = np.empty(n, dtype=np.int32)
    lib().s2vo_degrees(n, _p(row_ptr), _p(cols), _p(sol), _p(out))
    return out


def embed(row_ptr, cols, sol, theta: dict, num_layers: int, dtype=np.float32) -> np.ndarray:
    """(n, K) node-major embedding after num_layers rounds."""
    n = len(row_ptr) - 1
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int32)
    sol = np.ascontiguousarray(sol, dtype=np.uint8)
    t = {k: np.ascontiguousarray(v, dtype=dtype) for k, v in theta.items()}
    K = t["theta1"].shape[0]
    out = np.empty((n, K), dtype=dtype)
    rc = getattr(lib(), f"s2vo_embed_{_suffix(dtype)}")(
        n, _p(row_ptr), _p(cols), _p(sol), _p(t["theta1"]), _p(t["theta2"]),
        _p(t["theta3"]), _p(t["theta4"]), K, num_layers, _p(out))
    if rc:
        raise MemoryError("oracle embed failed")
    return out


def colsum(h: np.ndarray) -> np.ndarray:
    h = np.ascontiguousarray(h)
    n, K = h.shape
    g = np.empty(K, dtype=h.dtype)
    getattr(lib(), f"s2vo_colsum_{_suffix(h.dtype)}")(n, K, _p(h), _p(g))
    return g


def scores(h: np.ndarray, cand, theta: dict, u1) -> np.ndarray:
    h = np.ascontiguousarray(h)
    n, K = h.shape
    dt = h.dtype
    cand = np.ascontiguousarray(cand, dtype=np.uint8)
    t6 = np.ascontiguousarray(theta["theta6"], dtype=dt)
    t7 = np.ascontiguousarray(theta["theta7"], dtype=dt)
    u1 = np.ascontiguousarray(u1, dtype=dt)
    out = np.empty(n, dtype=dt)
    getattr(lib(), f"s2vo_scores_{_suffix(dt)}")(n, K, _p(h), _p(cand), _p(t6), _p(t7),
                                                  _p(u1), _p(out))
    return out


def forward(row_ptr, cols, sol, theta: dict, num_layers: int, dtype=np.float32):
    """Embedding, g, u1 (numpy, as the reference computes it) and raw scores
    for one graph, with cand = residual degree > 0 and not in the solution."""
    h = embed(row_ptr, cols, sol, theta, num_layers, dtype)
    g = colsum(h)
    # pkg/src/graphrl/policy.py:201 -- (B,K) @ theta5.T, done with numpy as the
    # reference does (B=1 here)
    u1 = (g[None, :] @ np.asarray(theta["theta5"], dtype=dtype).T)[0]
    deg = degrees(row_ptr, cols, sol)
    cand = ((deg > 0) & (np.asarray(sol) == 0)).astype(np.uint8)
    sc = scores(h, cand, theta, u1)
    return h, g, u1, cand, sc


def generate_ba_edges(n: int, d: int, seed: int) -> np.ndarray:
    """graphrl.generate_ba(n, d, seed).edge_array via the C restatement
    (ba_oracle.c, graphs.py:125-157); used by bench.py's reference arm to
    build its input graph without the product library."""
    build()
    L = ctypes.CDLL(str(HERE / "libba_oracle.so"))
    L.s2vo_generate_ba.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_void_p]
    L.s2vo_generate_ba.restype = ctypes.c_int64
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    words = np.array([s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]),
                      int(st["uinteger"])], dtype=np.uint64)
    num = L.s2vo_generate_ba(n, d, words.ctypes.data, None)
    if num < 0:
        raise ValueError(f"generate_ba({n}, {d}) out of range")
    edges = np.empty((num, 2), dtype=np.int64)
    if L.s2vo_generate_ba(n, d, words.ctypes.data, edges.ctypes.data) != num:
        raise RuntimeError("oracle BA generator failed")
    return edges
