"""structure2vec-DQN policy: parameters, forward, exact gradients, Adam.

API mirrors pkg/src/graphrl/policy.py.  Numerics run in libs2v (sm_100a):

* embed_forward  -> s2v_e12_table + L x s2v_embed_round (+ halo all-gather of
  the new rows over NCCL between rounds when P > 1);
* q_forward      -> s2v_colsum (numpy pairwise order) + u1 = g @ theta5.T +
  s2v_score;
* loss_and_gradients / adam_step -> s2v_layer_backward, s2v_gather,
  s2v_head_backward, s2v_param_grads, s2v_adam.

Results are bit-identical to the reference's fp32 forward:
embeddings, Q-values and selections match the CPU oracle exactly at any P.
u1 = g @ theta5.T (B x K by K x K, 4K*B flops) is computed on the host with
numpy, in the reference's own BLAS call, because OpenBLAS' small-matrix/gemv
accumulation order for it is not a simple chain; it costs one
256-byte round trip per evaluation.
"""
from __future__ import annotations

import ctypes
import os
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _lib
from .device import ptr, stream_ptr
from .errors import DataError
from .state import PartitionedState

PARAM_NAMES = ("theta1", "theta2", "theta3", "theta4", "theta5", "theta6", "theta7")

_CKPT_MAGIC = b"GRLP"
_CKPT_VERSION = 1
_DTYPE_CODES = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}
_CODE_DTYPES = {v: k for k, v in _DTYPE_CODES.items()}


def param_shapes(k: int) -> dict[str, tuple[int, int]]:
    return {"theta1": (k, 1), "theta2": (k, 1), "theta3": (k, k), "theta4": (k, k),
            "theta5": (k, k), "theta6": (k, k), "theta7": (2 * k, 1)}


@dataclass
class PolicyParams:
    """The seven trainable matrices plus depth L (policy.py:43-113)."""
    theta1: np.ndarray
    theta2: np.ndarray
    theta3: np.ndarray
    theta4: np.ndarray
    theta5: np.ndarray
    theta6: np.ndarray
    theta7: np.ndarray
    num_layers: int

    @property
    def embed_dim(self) -> int:
        return self.theta1.shape[0]

    @property
    def dtype(self) -> np.dtype:
        return self.theta1.dtype

    def __post_init__(self):
        self.validate()

    def validate(self) -> None:
        expected = param_shapes(self.theta1.shape[0])
        for name in PARAM_NAMES:
            arr = getattr(self, name)
            if arr.shape != expected[name]:
                raise ValueError(f"{name} must have shape {expected[name]}, got {arr.shape}")
            if not np.all(np.isfinite(arr)):
                raise ValueError(f"{name} contains non-finite entries")
        if self.num_layers < 1:
            raise ValueError(f"num_layers must be >= 1, got {self.num_layers}")

    @classmethod
    def initialize(cls, embed_dim: int, num_layers: int, seed: int, scale: float = 0.05,
                   dtype=np.float32, orientation: str = "positive") -> "PolicyParams":
        """Seeded uniform init with the reference's draw order (policy.py:79-102)."""
        if orientation not in ("positive", "symmetric"):
            raise ValueError(f"unknown init orientation {orientation!r}")
        rng = np.random.default_rng(seed)
        shapes = param_shapes(embed_dim)
        arrays = {name: rng.uniform(-scale, scale, shapes[name]).astype(dtype)
                  for name in PARAM_NAMES}
        if orientation == "positive":
            arrays["theta6"] = np.abs(arrays["theta6"])
            arrays["theta7"][embed_dim:] = np.abs(arrays["theta7"][embed_dim:])
        return cls(num_layers=num_layers, **arrays)

    def astype(self, dtype) -> "PolicyParams":
        return PolicyParams(num_layers=self.num_layers,
                            **{n: getattr(self, n).astype(dtype) for n in PARAM_NAMES})

    def copy(self) -> "PolicyParams":
        return self.astype(self.dtype)

    def as_dict(self) -> dict[str, np.ndarray]:
        return {name: getattr(self, name) for name in PARAM_NAMES}


def zero_grads(params: PolicyParams) -> dict[str, np.ndarray]:
    return {name: np.zeros_like(getattr(params, name)) for name in PARAM_NAMES}


def flatten_arrays(arrays: dict[str, np.ndarray]) -> np.ndarray:
    return np.concatenate([arrays[name].ravel() for name in PARAM_NAMES])


def unflatten_arrays(vec: np.ndarray, k: int) -> dict[str, np.ndarray]:
    out, off = {}, 0
    for name, shp in param_shapes(k).items():
        size = shp[0] * shp[1]
        out[name] = vec[off:off + size].reshape(shp).copy()
        off += size
    return out


def _dt_code(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return _lib.S2V_F32
    if dt == np.float64:
        return _lib.S2V_F64
    raise ValueError(f"unsupported dtype {dt}")


def _torch_dtype(dtype):
    return torch.float32 if np.dtype(dtype) == np.float32 else torch.float64


class _DeviceParams:
    """The seven thetas packed in one device buffer.  Re-uploaded only when the
    host arrays changed (compared by value), so a solve loop uploads once."""

    _cache: dict = {}

    def __new__(cls, params: PolicyParams, device):
        flat = np.ascontiguousarray(flatten_arrays(params.as_dict()), dtype=params.dtype)
        key = (id(params), str(device))
        hit = cls._cache.get(key)
        if hit is not None and hit._flat.shape == flat.shape and hit._flat.dtype == flat.dtype \
                and np.array_equal(hit._flat, flat) and hit._owner() is params:
            return hit
        obj = super().__new__(cls)
        obj._init(params, device, flat)
        if len(cls._cache) > 64:
            cls._cache.clear()
        cls._cache[key] = obj
        return obj

    def __init__(self, params: PolicyParams, device):
        pass

    def _init(self, params: PolicyParams, device, flat):
        import weakref
        self._owner = weakref.ref(params)
        self._flat = flat.copy()
        self.buf = torch.from_numpy(flat).to(device, non_blocking=False)
        self.k = params.embed_dim
        self.offsets = {}
        off = 0
        for name, shp in param_shapes(self.k).items():
            self.offsets[name] = off
            off += shp[0] * shp[1]
        self.elem = flat.dtype.itemsize

    def ptr(self, name: str) -> int:
        return self.buf.data_ptr() + self.offsets[name] * self.elem


def _np_dtype(t: torch.dtype) -> np.dtype:
    return {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64),
            torch.int32: np.dtype(np.int32), torch.int64: np.dtype(np.int64),
            torch.uint8: np.dtype(np.uint8)}[t]


def _check_dtype(state: PartitionedState, params: PolicyParams) -> None:
    if np.dtype(params.dtype) not in _DTYPE_CODES:
        raise ValueError(f"unsupported parameter dtype {params.dtype}")


class DeviceEmbedding:
    """Lazy (B, K, rows) view of embeddings resident in HBM.

    Layout on device: node-major [B][P][rows_max][K]; materialised on the host
    (numpy, reference layout) only when a caller reads it.
    """

    def __init__(self, state: PartitionedState, h: torch.Tensor, k: int, dtype,
                 gathered: bool):
        self.state = state
        self.h = h
        self.k = k
        self.dtype = np.dtype(dtype)
        self.gathered = gathered
        self.shape = (state.batch, k, state.part.num_rows)
        self.ndim = 3

    def local_rows(self) -> torch.Tensor:
        st = self.state
        v = self.h.view(st.batch, st.world, st.rows_max, self.k)
        return v[:, st.part.rank, :st.part.num_rows, :]

    def __array__(self, dtype=None, copy=None):
        arr = self.local_rows().to("cpu").numpy().transpose(0, 2, 1)
        arr = np.ascontiguousarray(arr)
        return arr.astype(dtype) if dtype is not None else arr

    def __getitem__(self, idx):
        return np.asarray(self)[idx]

    def __len__(self):
        return self.shape[0]


def _buffers(state: PartitionedState, k: int, dtype, count: int):
    n_el = state.batch * state.world * state.rows_max * k
    tdt = _torch_dtype(dtype)

    def make():
        # P = 1: every round writes every row before anything reads it (no
        # padding rows), so no zero-fill pass over the buffers is needed
        alloc = torch.empty if state.world == 1 else torch.zeros
        return [alloc(n_el, dtype=tdt, device=state.device) for _ in range(count)]
    return state.workspace(f"h{count}", (k, np.dtype(dtype).str, count), make)


def _peer_list(state: PartitionedState, dc, name: str, t: torch.Tensor, as_array: bool):
    """Peer addresses of a workspace buffer, registered once per workspace
    (a collective on every rank at the same point)."""
    if not getattr(dc, "supports_push", False):
        return None
    # key by a registration generation stamped on the tensor object, not by
    # its address: every rank (re)allocates its workspaces at the same
    # points, so the generations agree across ranks, while a reused address
    # on one rank only would desynchronise the peers_of collective
    gen = getattr(t, "_s2v_peer_gen", None)
    if gen is None:
        gen = state._peer_gen = getattr(state, "_peer_gen", 0) + 1
        t._s2v_peer_gen = gen
    key = (gen, t.numel(), as_array)
    return state.workspace(f"peers:{name}", key,
                           lambda: dc.peer_array(t) if as_array else dc.peers_of(t))


def _allgather_rows(state: PartitionedState, comm, h: torch.Tensor, k: int, tag: str,
                    name: str = ""):
    """In-place halo all-gather of every slot's rank chunk (device transport)."""
    if state.world == 1:
        return
    dc = comm.device_comm()
    chunk = state.rows_max * k * h.element_size()
    peers = _peer_list(state, dc, name or tag, h, False)
    dc.allgather_rows(h, chunk, chunk * state.world, state.batch, stream_ptr(), peers=peers)
    comm.record(tag, state.rows_max * k * state.batch)


# bench hook: when a list, every round that gathers neighbour rows of the
# previous round from HBM appends (start, end) CUDA events recorded on the
# launching stream around its kernel (the degree-table round 2 is not one)
ROUND_TIMER = None
# bench hook: when a list, loss_and_gradients appends (tag, start, end) around
# every s2v_layer_backward (tag: ("layer_backward", first, has_m, has_dm)) and
# s2v_gather (("gather",)) launch
BWD_TIMER = None


def _degree_table_round2(state: PartitionedState, k: int, dt: int, num_layers: int,
                         tape: bool = False) -> bool:
    """Round 2 from the per-degree table of round-1 outputs (s2v_h1_table +
    s2v_embed_round2_table): K = 64 fp32; at P > 1 for inference (the ranks
    exchange 4-byte residual degrees instead of 256-byte h1 rows).
    S2V_DEG_TABLE=0 turns it off (the plain round reading h1 gives the same
    bits)."""
    return (k == 64 and dt == _lib.S2V_F32 and num_layers >= 2
            and (state.world == 1 or not tape)
            and os.environ.get("S2V_DEG_TABLE", "1") != "0")


def _forward_rounds(state: PartitionedState, dparams: _DeviceParams, num_layers: int, comm,
                    dtype, tape: bool, reuse_tables: bool = False, persist: bool = False,
                    round_rows=None):
    """L embedding rounds.  Returns the list of h buffers (all of them when
    tape, else the final one) and, when tape, the m buffers per round.
    reuse_tables: the e12 / h1 tables of this state were last built from
    these same device parameters (an episode's later evaluations) -- skip
    rebuilding them.  persist: one buffer per layer (not ping-pong), so that
    every layer's rows survive to the next evaluation (incremental forward).
    round_rows(layer) -> (row list, active_n pair) device pointers: round
    layer+1 visits only those rows (the incremental frontier, full CSR)."""
    k = dparams.k
    dt = _dt_code(dtype)
    st = stream_ptr()
    max_deg = int(state.max_deg)
    table = state.workspace("e12", (k, np.dtype(dtype).str, max_deg), lambda: torch.empty(
        (max_deg + 2) * k, dtype=_torch_dtype(dtype), device=state.device))
    reuse = reuse_tables and getattr(state, "_tables_of", None) is dparams
    if not reuse:
        _lib.call("s2v_e12_table", dt, dparams.ptr("theta1"), dparams.ptr("theta2"),
                  dparams.ptr("theta3"), k, max_deg, ptr(table), st)
    if tape or persist:
        hs = _buffers(state, k, dtype, num_layers)
    else:
        hs = _buffers(state, k, dtype, 2)
    ms = None
    if tape:
        rows = state.batch * state.part.num_rows
        ms = state.workspace("mtape", (k, np.dtype(dtype).str, num_layers), lambda: [
            torch.empty(max(rows * k, 1), dtype=_torch_dtype(dtype), device=state.device)
            for _ in range(num_layers)])
    h_prev = None
    out = []
    h1t = None
    if _degree_table_round2(state, k, dt, num_layers, tape):
        h1t = state.workspace("h1t", (k, max_deg), lambda: torch.empty(
            (max_deg + 2) * k, dtype=torch.float32, device=state.device))
        if not reuse:
            _lib.call("s2v_h1_table", dt, dparams.ptr("theta4"), ptr(table), k, max_deg,
                      ptr(h1t), st)
    elif state.active_on:
        raise RuntimeError("active-row lists need the degree-table round (K = 64 fp32)")
    state._tables_of = dparams
    sh = state.shard
    outer = (sh.active, sh.active_n, sh.active_ptr, sh.active_cols)
    for layer in range(num_layers):
        h_out = hs[layer] if (tape or persist) else hs[layer % 2]
        m_out = ms[layer] if (tape and layer > 0) else None
        if round_rows is not None and layer > 0:
            rows_ptr, n_ptr = round_rows(layer)
            sh.active, sh.active_n, sh.active_ptr, sh.active_cols = rows_ptr, n_ptr, None, None
        if h1t is not None and layer == 0 and not tape:
            # inference: nothing reads h1 but round 2, which reads the table
            out.append(None)
            continue
        if h1t is not None and layer == 1:
            deg = None
            peers = None
            dc = comm.device_comm() if state.world > 1 else None
            if dc is not None:
                # every rank's residual degrees by physical row (4 B per node
                # instead of the 256-byte h1 rows a plain round 2 gathers)
                deg = state.workspace("trow", state.batch * state.world * state.rows_max,
                                      lambda: torch.zeros(
                                          max(state.batch * state.world * state.rows_max, 1),
                                          dtype=torch.int32, device=state.device))
                _lib.call("s2v_trow", state.shard_ref(), max_deg, ptr(deg), st)
                _allgather_rows(state, comm, deg, 1, "trow", name="trow")
                if dc.supports_push:
                    peers = _peer_list(state, dc, f"h{layer % 2}/{len(hs)}", h_out, True)
            _lib.call("s2v_embed_round2_table", dt, state.shard_ref(), dparams.ptr("theta4"),
                      ptr(table), k, max_deg, ptr(h1t), ptr(deg), ptr(h_out), ptr(peers),
                      state.world if peers is not None else 0, ptr(m_out), st)
            if dc is not None:
                if peers is not None:
                    dc.signal_and_wait(st)
                    comm.record("embed_fwd", state.rows_max * k * state.batch)
                else:
                    _allgather_rows(state, comm, h_out, k, "embed_fwd",
                                    name=f"h{layer % 2}/{len(hs)}")
            sh.active, sh.active_n, sh.active_ptr, sh.active_cols = outer
            h_prev = h_out
            out.append(h_out)
            continue
        timer = ROUND_TIMER if (ROUND_TIMER is not None and h_prev is not None) else None
        if timer is not None:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record()
        dc = comm.device_comm() if state.world > 1 else None
        if dc is not None and dc.supports_push and k == 64 and dt == _lib.S2V_F32:
            # fused halo exchange: the kernel stores each row into every peer
            peers = _peer_list(state, dc,
                               f"h{layer if (tape or persist) else layer % 2}/{len(hs)}", h_out,
                               True)
            _lib.call("s2v_embed_round_peers", dt, state.shard_ref(), dparams.ptr("theta4"),
                      ptr(table), k, max_deg, ptr(h_prev), ptr(h_out), ptr(peers), state.world,
                      ptr(m_out), st)
            dc.signal_and_wait(st)
            comm.record("embed_fwd", state.rows_max * k * state.batch)
        else:
            _lib.call("s2v_embed_round", dt, state.shard_ref(), dparams.ptr("theta4"),
                      ptr(table), k, max_deg, ptr(h_prev), ptr(h_out), ptr(m_out), st)
            _allgather_rows(state, comm, h_out, k, "embed_fwd",
                            name=f"h{layer if (tape or persist) else layer % 2}/{len(hs)}")
        sh.active, sh.active_n, sh.active_ptr, sh.active_cols = outer
        if timer is not None:
            ev1.record()
            timer.append((ev0, ev1))
        h_prev = h_out
        out.append(h_out)
    return out, ms, table


def embed_forward(state: PartitionedState, params: PolicyParams, comm) -> DeviceEmbedding:
    """(B, K, rows) embeddings of the locally owned nodes (policy.py:182-185)."""
    _check_dtype(state, params)
    dparams = _DeviceParams(params, state.device)
    hs, _, _ = _forward_rounds(state, dparams, params.num_layers, comm, params.dtype, False)
    # a fresh buffer, like the reference's freshly allocated result (the
    # workspace is reused by the next forward on this state)
    return DeviceEmbedding(state, hs[-1].clone(), params.embed_dim, params.dtype, gathered=True)


def _as_device_embedding(embed, state_hint, params: PolicyParams, comm) -> DeviceEmbedding:
    if isinstance(embed, DeviceEmbedding):
        return embed
    raise TypeError("q_forward needs the DeviceEmbedding returned by embed_forward")


def _colsum_device(emb: DeviceEmbedding) -> torch.Tensor:
    """g = pairwise sum over all N nodes of every slot (policy.py:199-200),
    left on the device ([B][K])."""
    st = emb.state
    k = emb.k
    lib = _lib.load()
    wsb = max(lib.s2v_colsum_workspace(st.shard_ref(), k, emb.dtype.itemsize),
              lib.s2v_colsum_residual_workspace(st.shard_ref(), k, emb.dtype.itemsize))
    ws = st.workspace("colsum", (k, emb.dtype.str), lambda: {
        "ws": torch.empty(max(wsb // emb.dtype.itemsize, 1), dtype=_torch_dtype(emb.dtype),
                          device=st.device),
        "g": torch.empty(st.batch * k, dtype=_torch_dtype(emb.dtype), device=st.device)})
    if st.active_on:
        # rows off the active list were never written this forward: they
        # take their (constant) round-1 row from the h1 table; an episode
        # keeps its own tree workspace so that all-dead leaves are reused
        h1t = st.workspace("h1t", (k, int(st.max_deg)), None)
        # P > 1: every rank's e12 rows by physical row, exchanged by this
        # forward's round 2, classify the gathered buffer's rows
        trow = st._ws["trow"][1] if st.world > 1 else None
        inc = st.colsum_cache
        if inc is None:
            _lib.call("s2v_colsum_residual", _dt_code(emb.dtype), st.shard_ref(), k, ptr(emb.h),
                      ptr(h1t), int(st.max_deg), ptr(ws["g"]), ptr(ws["ws"]), wsb, None, 1,
                      None, None, ptr(trow), stream_ptr())
        else:
            if inc.get("ws") is None:
                inc["ws"] = torch.empty_like(ws["ws"])
                inc["last"] = torch.zeros(st.batch * st.num_nodes, dtype=torch.uint8,
                                          device=st.device)
            # incremental forward: (rows, count) whose embedding changed
            dirty = inc.get("dirty") or (None, None)
            _lib.call("s2v_colsum_residual", _dt_code(emb.dtype), st.shard_ref(), k, ptr(emb.h),
                      ptr(h1t), int(st.max_deg), ptr(ws["g"]), ptr(inc["ws"]), wsb,
                      ptr(inc["last"]), 1 if inc["full"] else 0, dirty[0], dirty[1],
                      ptr(trow), stream_ptr())
            inc["full"] = False
    else:
        _lib.call("s2v_colsum", _dt_code(emb.dtype), st.shard_ref(), k, ptr(emb.h),
                  ptr(ws["g"]), ptr(ws["ws"]), wsb, stream_ptr())
    return ws["g"]


def _global_sum(emb: DeviceEmbedding) -> np.ndarray:
    return _colsum_device(emb).to("cpu").numpy().reshape(emb.state.batch, emb.k)


def u1_on_device(batch: int, k: int, dtype) -> bool:
    """Whether libs2v reproduces numpy's g @ theta5.T order for this shape."""
    return np.dtype(dtype) == np.float32 and bool(_lib.load().s2v_u1_exact(batch, k))


def score_workspace(st: PartitionedState, k: int, dtype) -> dict:
    """Device buffers of the scorer: u1, scores, per-block keys, the read-back
    vector (counts [B] then top keys [B][8][2]) and a candidate override."""
    dtype = np.dtype(dtype)
    nblk = _lib.load().s2v_score_blocks(st.shard_ref())
    rows = st.batch * st.part.num_rows
    return st.workspace("score", (k, dtype.str), lambda: {
        "u1": torch.empty(st.batch * k, dtype=_torch_dtype(dtype), device=st.device),
        "scores": torch.empty(max(rows, 1), dtype=_torch_dtype(dtype), device=st.device),
        "bkeys": torch.empty(st.batch * nblk * 8 * 2, dtype=torch.int64, device=st.device),
        "out": torch.empty(st.batch * (1 + 8 * 2), dtype=torch.int64, device=st.device),
        "cand": torch.empty(max(rows, 1), dtype=torch.uint8, device=st.device)})


def _score(emb: DeviceEmbedding, params: PolicyParams, dparams: _DeviceParams,
           cand_override: np.ndarray | None, mode: int, d: int, readback: bool = True):
    """Run the scorer; returns (scores device tensor, top keys (B,d,2) or None,
    counts (B,))."""
    st = emb.state
    k = emb.k
    device_u1 = u1_on_device(st.batch, k, emb.dtype)
    if not device_u1:
        g = _global_sum(emb)
        # policy.py:201 -- the reference's own numpy product, on the host
        u1 = np.ascontiguousarray(g @ params.theta5.T, dtype=params.dtype)
    rows = st.batch * st.part.num_rows
    ws = score_workspace(st, k, emb.dtype)
    if device_u1:  # numpy's own accumulation order, reproduced on device
        _lib.call("s2v_u1", _dt_code(emb.dtype), st.batch, k, ptr(_colsum_device(emb)),
                  dparams.ptr("theta5"), ptr(ws["u1"]), stream_ptr())
    else:
        ws["u1"].copy_(torch.from_numpy(u1.reshape(-1)))
    cand_ptr = None
    if cand_override is not None:
        ws["cand"][:rows].copy_(torch.from_numpy(
            np.ascontiguousarray(cand_override, dtype=np.uint8).reshape(-1)))
        cand_ptr = ptr(ws["cand"])
    s = stream_ptr()
    _lib.call("s2v_score", _dt_code(emb.dtype), st.shard_ref(), k, ptr(emb.h), ptr(ws["u1"]),
              dparams.ptr("theta6"), dparams.ptr("theta7"), cand_ptr, mode,
              ptr(ws["scores"]), ptr(ws["bkeys"]), ptr(ws["out"]), s)
    top = None
    if d > 0:
        _lib.call("s2v_topk_merge", st.shard_ref(), ptr(ws["bkeys"]), min(d, _lib.TOPK_MAX),
                  ws["out"].data_ptr() + 8 * st.batch, s)
    if not readback:
        return ws
    out = ws["out"].to("cpu").numpy()  # counts and keys in one read-back
    counts = out[:st.batch].copy()
    if d > 0:
        dm = min(d, _lib.TOPK_MAX)
        top = out[st.batch:st.batch + st.batch * dm * 2].view(np.uint64).reshape(st.batch, dm, 2)
        if d > _lib.TOPK_MAX:
            top = _more_keys(st, ws, cand_ptr, mode, top.copy(), d)
    return ws["scores"][:rows], top, counts


def _more_keys(st: PartitionedState, ws, cand_ptr, mode: int, top: np.ndarray, d: int):
    """Top-d for d > 8 (SelectionSchedule.fixed(d) allows any d): per-row keys
    once, then repeated top-8 passes strictly below the last key taken."""
    rows = st.batch * st.part.num_rows
    kw = st.workspace("keys_all", rows, lambda: {
        "keys": torch.empty(max(rows, 1) * 2, dtype=torch.int64, device=st.device),
        "ceil": torch.empty(st.batch * 2, dtype=torch.int64, device=st.device),
        "top": torch.empty(st.batch * 8 * 2, dtype=torch.int64, device=st.device)})
    s = stream_ptr()
    fn = "s2v_score_keys" if ws["scores"].dtype == torch.float32 else "s2v_score_keys_f64"
    _lib.call(fn, st.shard_ref(), ptr(ws["scores"]), cand_ptr or ptr(st.cand_d), mode,
              ptr(kw["keys"]), s)
    parts = [top]
    have = top.shape[1]
    while have < d:
        last = parts[-1][:, -1, :]
        if not np.any(last[:, 0]):  # every slot exhausted
            break
        kw["ceil"].copy_(torch.from_numpy(np.ascontiguousarray(last).view(np.int64).reshape(-1)))
        _lib.call("s2v_topk_below", st.shard_ref(), ptr(kw["keys"]), ptr(kw["ceil"]),
                  ptr(ws["bkeys"]), s)
        _lib.call("s2v_topk_merge", st.shard_ref(), ptr(ws["bkeys"]), 8, ptr(kw["top"]), s)
        nxt = kw["top"].to("cpu").numpy().view(np.uint64).reshape(st.batch, 8, 2).copy()
        nxt[last[:, 0] == 0] = 0  # a slot already exhausted stays empty
        parts.append(nxt)
        have += 8
    return np.concatenate(parts, axis=1)[:, :d]


def q_forward(embed, cand: np.ndarray, params: PolicyParams, comm) -> np.ndarray:
    """(B, rows) scores for every locally owned node (policy.py:214-218).
    `cand` is the sparse-diagonal extractor (non-candidates get a zeroed
    own-embedding term); masking happens in masked_scores."""
    emb = _as_device_embedding(embed, None, params, comm)
    st = emb.state
    dparams = _DeviceParams(params, st.device)
    cand = np.asarray(cand)
    override = None if cand is st.cand else cand
    comm.record("q_fwd", st.batch * emb.k)
    scores, _, _ = _score(emb, params, dparams, override, 0, 0)
    return scores.to("cpu").numpy().reshape(st.batch, st.part.num_rows).astype(params.dtype)


def masked_scores(scores: np.ndarray, cand: np.ndarray) -> np.ndarray:
    """Scores with non-candidates pushed to -inf (policy.py:221-224)."""
    neg = np.array(-np.inf, dtype=scores.dtype)
    return np.where(cand.astype(bool), scores, neg)


def decode_keys(top: np.ndarray):
    """(..., 2) uint64 keys -> (node ids int64, scores float64, valid bool)."""
    s = top[..., 0]
    node = (~top[..., 1]).astype(np.int64)
    valid = s != 0
    sign = np.uint64(1) << np.uint64(63)
    bits = np.where(s & sign, s & ~sign, ~s)
    vals = bits.view(np.float64).copy()
    vals[s == np.uint64(0xFFFFFFFFFFFFFFFF)] = np.nan
    return node, vals, valid


def evaluate_device(state: PartitionedState, params: PolicyParams, dparams, comm, d: int,
                    mode: int = 0, reuse_tables: bool = False):
    """evaluate() without any host round trip (P = 1, device u1): returns the
    score workspace whose "out" holds counts [B] then top-d keys [B][d][2]."""
    hs, _, _ = _forward_rounds(state, dparams, params.num_layers, comm, params.dtype, False,
                               reuse_tables=reuse_tables)
    emb = DeviceEmbedding(state, hs[-1], params.embed_dim, params.dtype, gathered=True)
    return _score(emb, params, dparams, None, mode, d, readback=False)


def merge_rank_keys(top: np.ndarray, counts: np.ndarray, comm, d: int):
    """Merge every rank's top-d keys (B, d, 2) and candidate counts into the
    global top-d, identically on every rank (replaces the reference's
    all_gather of the full (B, N) score matrix, inference.py:113).  Keys
    order by score image then ~node, so the merge keeps descending score
    with lowest-index ties."""
    b = top.shape[0]
    keys = comm.all_gather(top.reshape(b, -1), axis=-1, tag="select").reshape(b, -1, 2)
    counts = comm.all_reduce_sum(counts, tag="select")
    order = np.lexsort((keys[..., 1], keys[..., 0]), axis=-1)[:, ::-1][:, :d]
    return np.take_along_axis(keys, order[..., None], axis=1), counts


def evaluate(state: PartitionedState, params: PolicyParams, comm, d: int, mode: int = 0):
    """Fused policy evaluation for the selection loops: embed + score + top-d
    keys, nothing but keys and counts leave the device.  Returns
    (nodes (B,d), scores (B,d), valid (B,d), counts (B,))."""
    dparams = _DeviceParams(params, state.device)
    hs, _, _ = _forward_rounds(state, dparams, params.num_layers, comm, params.dtype, False)
    emb = DeviceEmbedding(state, hs[-1], params.embed_dim, params.dtype, gathered=True)
    _, top, counts = _score(emb, params, dparams, None, mode, d)
    if state.world > 1:
        top, counts = merge_rank_keys(top, counts, comm, d)
    nodes, vals, valid = decode_keys(top)
    return nodes, vals, valid, counts


# ---------------------------------------------------------------------------
# Loss and exact gradients (policy.py:232-315)
# ---------------------------------------------------------------------------


def loss_and_gradients(state: PartitionedState, actions, targets, params: PolicyParams, comm):
    """MSE of Q(s_t, a_t) against targets with exact gradients.

    Forward with tape (all h_l, m_l resident in HBM), Q head at the action
    nodes on their owner rank, dg exchange, L-1 backward rounds (dm halo
    exchange + alive-neighbour gather), theta1..theta4 reductions, one fp64
    gradient pack (identical on every rank).  Returns (loss, grads)."""
    b, n = state.batch, state.num_nodes
    k = params.embed_dim
    dtype = np.dtype(params.dtype)
    actions = np.asarray(actions, dtype=np.int64)
    targets = np.asarray(targets, dtype=dtype)
    if actions.shape != (b,) or targets.shape != (b,):
        raise ValueError(f"need {b} actions and targets, got {actions.shape} and {targets.shape}")
    if not np.all(np.isfinite(targets)):
        raise ValueError("targets must be finite")
    if np.any(actions < 0) or np.any(actions >= n):
        raise ValueError("action node index out of range")
    _check_dtype(state, params)
    pack = _loss_pack(state, actions, targets, params, _DeviceParams(params, state.device), comm)
    reduced = pack.to("cpu").numpy()
    grads = unflatten_arrays(reduced[:-1].astype(dtype), k)
    return float(reduced[-1]) / b, grads


def _loss_pack(state: PartitionedState, actions: np.ndarray, targets: np.ndarray,
               params: PolicyParams, dparams, comm) -> torch.Tensor:
    """loss_and_gradients on the device: the fp64 pack [grads in parameter
    order, summed squared error], identical on every rank; dparams holds the
    parameters the kernels read."""
    b = state.batch
    k = params.embed_dim
    dtype = np.dtype(params.dtype)
    dt = _dt_code(dtype)
    tdt = _torch_dtype(dtype)
    dev = state.device
    s = stream_ptr()
    L = params.num_layers
    lib = _lib.load()
    hs, ms, _ = _forward_rounds(state, dparams, L, comm, dtype, tape=True)
    comm.record("q_fwd", b * k)
    rows = state.batch * state.part.num_rows
    nblk = lib.s2v_backward_blocks(state.shard_ref())
    full = state.batch * state.world * state.rows_max * k
    head_len = 2 * k * k + 2 * k + 1
    plen = 2 * k + k * k
    ws = state.workspace("bwd", (k, dtype.str, L), lambda: {
        "actions": torch.empty(b, dtype=torch.int64, device=dev),
        "targets": torch.empty(b, dtype=tdt, device=dev),
        "head": torch.empty(b * head_len, dtype=torch.float64, device=dev),
        "dg": torch.empty(b * k, dtype=tdt, device=dev),
        "dact": torch.empty(b * k, dtype=tdt, device=dev),
        "grad_h": torch.empty(max(rows * k, 1), dtype=tdt, device=dev),
        "dzsum": torch.empty(max(rows * k, 1), dtype=tdt, device=dev),
        "dm": torch.zeros(full, dtype=tdt, device=dev),
        "p4": torch.empty(nblk * k * k, dtype=tdt, device=dev),
        "pp": torch.empty(nblk * plen, dtype=tdt, device=dev),
        "t2tot": torch.empty(b * k, dtype=tdt, device=dev),
        "pack": torch.empty(4 * k * k + 4 * k + 1, dtype=torch.float64, device=dev)})
    ws["actions"].copy_(torch.from_numpy(actions))
    ws["targets"].copy_(torch.from_numpy(np.ascontiguousarray(targets)))
    # g = pairwise sum of h_L (policy.py:199-200), kept on device
    emb = DeviceEmbedding(state, hs[-1], k, dtype, gathered=True)
    # the "colsum" workspace is shared with _colsum_device: sized for both
    wsb = max(lib.s2v_colsum_workspace(state.shard_ref(), k, dtype.itemsize),
              lib.s2v_colsum_residual_workspace(state.shard_ref(), k, dtype.itemsize))
    cs = state.workspace("colsum", (k, dtype.str), lambda: {
        "ws": torch.empty(max(wsb // dtype.itemsize, 1), dtype=tdt, device=dev),
        "g": torch.empty(b * k, dtype=tdt, device=dev)})
    _lib.call("s2v_colsum", dt, state.shard_ref(), k, ptr(emb.h), ptr(cs["g"]), ptr(cs["ws"]),
              wsb, s)
    _lib.call("s2v_head_backward", dt, state.shard_ref(), k, ptr(hs[-1]), ptr(cs["g"]),
              ptr(ws["actions"]), ptr(ws["targets"]), dparams.ptr("theta5"),
              dparams.ptr("theta6"), dparams.ptr("theta7"), ptr(ws["head"]), ptr(ws["dg"]),
              ptr(ws["dact"]), s)
    dc = comm.device_comm() if state.world > 1 else None
    if dc is not None:  # q_bwd: the adjoint of g reaches every rank's rows
        dc.allreduce(ptr(ws["dg"]), b * k, 2 if dtype == np.float32 else 1, s)
    comm.record("q_bwd", b * k)
    _lib.call("s2v_grad_h_init", dt, state.shard_ref(), k, ptr(ws["dg"]), ptr(ws["actions"]),
              ptr(ws["dact"]), ptr(ws["grad_h"]), s)
    timer = BWD_TIMER

    def timed(tag, fn):
        if timer is None:
            return fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        timer.append((tag, e0, e1))

    for layer in range(L - 1, -1, -1):
        last = layer == 0
        flags = (layer == L - 1, layer > 0, not last)  # first, m_l, dm_out
        timed(("layer_backward",) + flags, lambda: _lib.call(
            "s2v_layer_backward", dt, state.shard_ref(), k, dparams.ptr("theta4"),
            ptr(ws["grad_h"]), ptr(hs[layer]), ptr(ms[layer]) if layer > 0 else None,
            ptr(ws["dzsum"]), ptr(ws["p4"]), 1 if layer == L - 1 else 0,
            None if last else ptr(ws["dm"]), s))
        if last:
            break
        _allgather_rows(state, comm, ws["dm"], k, "embed_bwd", name="dm")
        timed(("gather",), lambda: _lib.call("s2v_gather", dt, state.shard_ref(), k,
                                             ptr(ws["dm"]), ptr(ws["grad_h"]), s))
    # dtheta2's einsum terms go to a chain-layout buffer: grad_h is free by
    # now and has the size unless K is not a multiple of 32 / itemsize
    t2b = lib.s2v_theta2_terms_bytes(dt, state.shard_ref(), k)
    t2c = ws["grad_h"] if t2b <= ws["grad_h"].numel() * dtype.itemsize else \
        state.workspace("theta2_terms", (t2b,), lambda: torch.empty(
            t2b // dtype.itemsize, dtype=tdt, device=dev))
    _lib.call("s2v_param_grads", dt, state.shard_ref(), k, dparams.ptr("theta2"),
              dparams.ptr("theta3"), ptr(ws["dzsum"]), ptr(ws["pp"]), ptr(t2c), s)
    pack = ws["pack"]
    base = pack.data_ptr()
    _lib.call("s2v_reduce_partials", dt, ptr(ws["pp"]), nblk, plen, base, s)  # t1, t2, t3
    # dtheta2 in the reference's einsum order (policy.py:305-306) replaces
    # the partial-sum value: the 4M-term sum cancels heavily at BA(2M,16)
    _lib.call("s2v_theta2_einsum", dt, state.shard_ref(), k, ptr(t2c), ptr(ws["t2tot"]),
              base + 8 * k, s)
    _lib.call("s2v_reduce_partials", dt, ptr(ws["p4"]), nblk, k * k, base + 8 * plen, s)
    _lib.call("s2v_reduce_partials", _lib.S2V_F64, ptr(ws["head"]), b, head_len,
              base + 8 * (plen + k * k), s)  # t5, t6, t7, sq_err
    if dc is not None:
        dc.allreduce(base, pack.numel(), 1, s)
    comm.record("grad", pack.numel())
    return pack


def train_iterations(state: PartitionedState, actions, targets, params: PolicyParams,
                     adam: "AdamState", tau: int, comm) -> list[float]:
    """tau x (loss_and_gradients + adam_step) of train_step (agent.py:252-260)
    with parameters, moments and gradients resident on the device: no host
    round trip inside the loop, one read-back at the end.  Same kernels and
    rounding as the host-driven loop; a non-finite gradient rejects that
    step and every later one (adam_step's rule) and raises its ValueError."""
    b, n = state.batch, state.num_nodes
    k = params.embed_dim
    dtype = np.dtype(params.dtype)
    actions = np.asarray(actions, dtype=np.int64)
    targets = np.asarray(targets, dtype=dtype)
    if actions.shape != (b,) or targets.shape != (b,):
        raise ValueError(f"need {b} actions and targets, got {actions.shape} and {targets.shape}")
    if not np.all(np.isfinite(targets)):
        raise ValueError("targets must be finite")
    if np.any(actions < 0) or np.any(actions >= n):
        raise ValueError("action node index out of range")
    _check_dtype(state, params)
    dev = state.device
    dparams = _DeviceParams(params, dev)
    tdt = _torch_dtype(dtype)
    m_d = torch.from_numpy(np.ascontiguousarray(flatten_arrays(adam.m), dtype=dtype)).to(dev)
    v_d = torch.from_numpy(np.ascontiguousarray(flatten_arrays(adam.v), dtype=dtype)).to(dev)
    npar = m_d.numel()
    bad = torch.zeros(max(tau, 1), dtype=torch.int32, device=dev)
    losses = torch.zeros(max(tau, 1), dtype=torch.float64, device=dev)
    pack = None
    for it in range(tau):
        pack = _loss_pack(state, actions, targets, params, dparams, comm)
        losses[it:it + 1].copy_(pack[-1:])
        step = adam.step + it + 1
        _lib.call("s2v_adam_pack", _dt_code(dtype), dparams.buf.data_ptr(), ptr(pack), ptr(m_d),
                  ptr(v_d), npar, adam.beta1, 1 - adam.beta1, adam.beta2, 1 - adam.beta2,
                  adam.eps, adam.lr, 1.0 - adam.beta1 ** step, 1.0 - adam.beta2 ** step,
                  ptr(bad), it, stream_ptr())
    if tau <= 0:
        return []
    # one read-back: flags, parameters, moments and losses as one byte buffer
    outs = (bad, dparams.buf, m_d, v_d, losses)
    raw = torch.cat([t.reshape(-1).view(torch.uint8) for t in outs]).to("cpu").numpy()
    parts, off = [], 0
    for t in outs:
        nb = t.numel() * t.element_size()
        parts.append(raw[off:off + nb].view(_np_dtype(t.dtype)))
        off += nb
    flags, new_p, m_h, v_h, loss_h = parts
    done = int(np.argmax(flags != 0)) if flags.any() else tau
    for name, arr in unflatten_arrays(new_p.astype(dtype), k).items():
        getattr(params, name)[...] = arr
    for name, arr in unflatten_arrays(m_h.copy(), k).items():
        adam.m[name] = arr
    for name, arr in unflatten_arrays(v_h.copy(), k).items():
        adam.v[name] = arr
    adam.step += done
    dparams._flat = np.ascontiguousarray(flatten_arrays(params.as_dict()), dtype=dtype)
    if done < tau:
        grads = unflatten_arrays(pack.to("cpu").numpy()[:-1].astype(dtype), k)
        name = next(nm for nm in PARAM_NAMES if not np.all(np.isfinite(grads[nm])))
        raise ValueError(f"non-finite gradient for {name}; step rejected")
    return [float(x) / b for x in loss_h[:tau]]


# ---------------------------------------------------------------------------
# Adam (policy.py:323-359)
# ---------------------------------------------------------------------------


@dataclass
class AdamState:
    """First/second moments and step counter (policy.py:323-336)."""
    m: dict
    v: dict
    step: int = 0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    lr: float = 1e-5

    @classmethod
    def create(cls, params: PolicyParams, lr: float = 1e-5) -> "AdamState":
        return cls(m=zero_grads(params), v=zero_grads(params), lr=lr)


def adam_step(params: PolicyParams, grads: dict, state: AdamState) -> None:
    """One bias-corrected Adam update in place, on the device (s2v_adam);
    non-finite gradients are rejected before any state changes."""
    for name in PARAM_NAMES:
        if not np.all(np.isfinite(grads[name])):
            raise ValueError(f"non-finite gradient for {name}; step rejected")
    dtype = np.dtype(params.dtype)
    from .device import current_device
    dev = current_device()
    state.step += 1
    b1c = 1.0 - state.beta1 ** state.step
    b2c = 1.0 - state.beta2 ** state.step
    k = params.embed_dim
    packs = [np.ascontiguousarray(flatten_arrays(d), dtype=dtype)
             for d in (params.as_dict(), grads, state.m, state.v)]
    buf = torch.from_numpy(np.concatenate(packs)).to(dev)
    n = packs[0].size
    e = dtype.itemsize
    p0 = buf.data_ptr()
    _lib.call("s2v_adam", _dt_code(dtype), p0, p0 + n * e, p0 + 2 * n * e, p0 + 3 * n * e, n,
              state.beta1, 1 - state.beta1, state.beta2, 1 - state.beta2, state.eps, state.lr,
              b1c, b2c, stream_ptr())
    out = buf.to("cpu").numpy()
    new_p = unflatten_arrays(out[:n], k)
    new_m = unflatten_arrays(out[2 * n:3 * n], k)
    new_v = unflatten_arrays(out[3 * n:4 * n], k)
    for name in PARAM_NAMES:
        getattr(params, name)[...] = new_p[name]
        state.m[name] = new_m[name]
        state.v[name] = new_v[name]


# ---------------------------------------------------------------------------
# Checkpoints (policy.py:367-407): format unchanged
# ---------------------------------------------------------------------------


def save_checkpoint(params: PolicyParams, path) -> None:
    path = Path(path)
    code = _DTYPE_CODES.get(np.dtype(params.dtype))
    if code is None:
        raise ValueError(f"unsupported checkpoint dtype {params.dtype}")
    with open(path, "wb") as fh:
        fh.write(_CKPT_MAGIC)
        fh.write(struct.pack("<III B", _CKPT_VERSION, params.embed_dim, params.num_layers, code))
        for name in PARAM_NAMES:
            fh.write(np.ascontiguousarray(getattr(params, name)).tobytes())


def load_checkpoint(path) -> PolicyParams:
    path = Path(path)
    if not path.exists():
        raise DataError(f"checkpoint not found: {path}")
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != _CKPT_MAGIC:
            raise DataError(f"{path}: not a policy checkpoint (magic {magic!r})")
        version, k, layers, code = struct.unpack("<III B", fh.read(13))
        if version != _CKPT_VERSION:
            raise DataError(f"{path}: unsupported checkpoint version {version}")
        if code not in _CODE_DTYPES:
            raise DataError(f"{path}: unknown dtype code {code}")
        dtype = _CODE_DTYPES[code]
        arrays = {}
        for name, shp in param_shapes(k).items():
            nbytes = shp[0] * shp[1] * dtype.itemsize
            buf = fh.read(nbytes)
            if len(buf) != nbytes:
                raise DataError(f"{path}: truncated checkpoint at {name}")
            arrays[name] = np.frombuffer(buf, dtype=dtype).reshape(shp).copy()
        if fh.read(1):
            raise DataError(f"{path}: trailing bytes after parameters")
    return PolicyParams(num_layers=layers, **arrays)
