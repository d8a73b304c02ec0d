"""Device-resident residual graph state (one rank's row shard of B graphs).

API mirrors pkg/src/graphrl/state.py (Partition, partition_rows,
PartitionedState, apply_action, is_covered).  Where the reference keeps a
scipy CSR whose removed entries are zeroed values, this keeps, in HBM:

* row_ptr int64 [B*rows+1] and cols uint32 [nnz]: the local rows of every
  slot, neighbour lists ascending, each entry holding the neighbour's physical
  row in the embedding layout [B][P][rows_max] with bit 31 = removed;
* the transpose lookup col_ptr/col_ent/col_row (state.py:115-122's
  _col_order/_col_ptr) used to remove column v on every rank;
* rdeg int32, sol/cand uint8, residual int64 [B].

The structure of each graph is uploaded once per device and reused by every
state built from it (tuples_to_graphs, batch_targets, env resets).  Host views
(sol, cand, local_residual, local_degrees) are cached D2H mirrors, refreshed
after every mutation.
"""
from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import current_device, ptr, stream_ptr, to_device
from .errors import InvalidActionError
from .graphs import Graph


@dataclass(frozen=True)
class Partition:
    """The block of node rows owned by one rank (state.py:20-33)."""
    rank: int
    num_workers: int
    row_start: int
    row_stop: int

    @property
    def num_rows(self) -> int:
        return self.row_stop - self.row_start

    def owns(self, node: int) -> bool:
        return self.row_start <= node < self.row_stop


def partition_rows(n: int, p: int) -> list[Partition]:
    """Balanced block partition of [0, n) over p ranks (state.py:36-53)."""
    if p < 1:
        raise ValueError(f"worker count must be >= 1, got {p}")
    if p > n:
        raise ValueError(f"more workers ({p}) than nodes ({n})")
    base, extra = divmod(n, p)
    parts, start = [], 0
    for rank in range(p):
        stop = start + base + (1 if rank < extra else 0)
        parts.append(Partition(rank, p, start, stop))
        start = stop
    return parts


def rows_max_of(n: int, p: int) -> int:
    return -(-n // p)


def phys_rows(n: int, p: int) -> np.ndarray:
    """Physical row (slot 0) of every global node: r*rows_max + (u - start_r)."""
    base, extra = divmod(n, p)
    u = np.arange(n, dtype=np.int64)
    big = extra * (base + 1)
    r = np.where(u < big, u // (base + 1), extra + (u - big) // max(base, 1))
    start = r * base + np.minimum(r, extra)
    return r * rows_max_of(n, p) + (u - start)


# -- per-(graph, device, partition) structure cache ---------------------------

class _ShardStructure:
    """One graph's local rows on one device: CSR + transpose lookup."""

    def __init__(self, graph: Graph, part: Partition, device: torch.device):
        n, p = graph.num_nodes, part.num_workers
        row_ptr_g, cols_g = graph.csr_arrays()
        lo, hi = int(row_ptr_g[part.row_start]), int(row_ptr_g[part.row_stop])
        rows = part.num_rows
        self.nnz = hi - lo
        self.rows = rows
        # over the whole graph: e12 / h1 tables are indexed by the residual
        # degree of neighbours that other ranks own
        self.max_deg_global = int(np.diff(row_ptr_g).max()) if n else 0
        # the rest is built on the device (s2v_shard_structure): physical
        # column ids, the column lookup (stable argsort by neighbour id) and
        # the descending-degree processing order (rows above the hub degree
        # go to the CTA-cooperative kernel)
        # (one-shot uploads: pageable copies -- page-locking 256 MB first costs
        # more than it saves)
        self.row_ptr = to_device(row_ptr_g[part.row_start:part.row_stop + 1] - lo, device)
        nbr = to_device(cols_g[lo:hi], device) if self.nnz else \
            torch.zeros(1, dtype=torch.int32, device=device)
        self.cols0 = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=device)
        self.col_ptr = torch.empty(n + 1, dtype=torch.int64, device=device)
        self.col_ent = torch.empty(max(self.nnz, 1), dtype=torch.int64, device=device)
        self.col_row = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=device)
        self.order = torch.empty(max(rows, 1), dtype=torch.int32, device=device)
        n_hub, max_deg = ctypes.c_int64(0), ctypes.c_int32(0)
        _lib.call("s2v_shard_structure", n, p, rows_max_of(n, p), rows, ptr(self.row_ptr),
                  ptr(nbr), self.nnz, ptr(self.cols0), ptr(self.col_ptr), ptr(self.col_ent),
                  ptr(self.col_row), ptr(self.order), ctypes.byref(n_hub),
                  ctypes.byref(max_deg), stream_ptr())
        self.n_hub = int(n_hub.value)
        self.max_deg = int(max_deg.value)


def _structure(graph: Graph, part: Partition, device: torch.device) -> _ShardStructure:
    per_graph = graph._device_cache
    key = (device.index, part.num_workers, part.rank)
    st = per_graph.get(key)
    if st is None:
        st = _ShardStructure(graph, part, device)
        per_graph[key] = st
    return st


def _assemble(dev, dtype: torch.dtype, total: int, segments) -> torch.Tensor:
    """dst[off + i] = src[skip + i] + add for segments (src, off, len, add[, skip])
    in one s2v_segment_copy launch."""
    out = torch.empty(max(total, 1), dtype=dtype, device=dev)
    elem = out.element_size()
    table = np.zeros((len(segments), 4), dtype=np.int64)
    for i, sg in enumerate(segments):
        src, off, n, add = sg[:4]
        skip = sg[4] if len(sg) > 4 else 0
        table[i] = (src.data_ptr() + skip * elem, off, n, add)
    longest = int(table[:, 2].max()) if len(segments) else 0
    if longest:
        segs = to_device(table.reshape(-1), dev, pinned=True)
        _lib.call("s2v_segment_copy", elem, ptr(segs), len(segments), longest, ptr(out),
                  stream_ptr())
    return out


class PartitionedState:
    """One rank's slice of state for a batch of B graphs with equal N
    (state.py:56-111), resident in HBM."""

    def __init__(self, graphs: list[Graph], part: Partition,
                 solutions: np.ndarray | None = None, dtype=np.float32,
                 graph_ids: list[int] | None = None):
        if not graphs:
            raise ValueError("need at least one graph")
        n = graphs[0].num_nodes
        if any(g.num_nodes != n for g in graphs):
            raise ValueError("all graphs in a batch must have the same node count")
        batch = len(graphs)
        self.part = part
        self.num_nodes = n
        self.batch = batch
        self.graph_ids = list(graph_ids) if graph_ids is not None else list(range(batch))
        self.dtype = np.dtype(dtype)
        if solutions is None:
            solutions = np.zeros((batch, n), dtype=np.uint8)
        else:
            solutions = np.asarray(solutions, dtype=np.uint8)
            if solutions.shape != (batch, n):
                raise ValueError(
                    f"solutions must be (B, N) = ({batch}, {n}), got {solutions.shape}")
        self.device = current_device()
        dev = self.device
        P = part.num_workers
        self.world = P
        self.rows_max = rows_max_of(n, P)
        rows = part.num_rows
        structs = [_structure(g, part, dev) for g in graphs]
        self.max_deg = max(s.max_deg_global for s in structs)
        ent_off = np.zeros(batch + 1, dtype=np.int64)
        np.cumsum([s.nnz for s in structs], out=ent_off[1:])
        self.nnz = int(ent_off[-1])
        slot_stride = P * self.rows_max
        if batch == 1 and self.nnz:
            # one slot: the cached read-only structure is used in place; only
            # the column array (which carries the removed-edge bits) is a
            # copy, written by s2v_shard_init from the structure's
            s0 = structs[0]
            self.row_ptr, self.col_ptr, self.col_ent, self.col_row = (
                s0.row_ptr, s0.col_ptr, s0.col_ent, s0.col_row)
            self.cols = torch.empty_like(s0.cols0)
            cols_src = s0.cols0
            self.order = s0.order if rows else torch.zeros(1, dtype=torch.int32, device=dev)
        else:
            # block-diagonal assembly over slots (device-to-device, structure
            # cached): one segment-copy launch per array
            cols_src = None
            e = [int(x) for x in ent_off]
            lp = int(structs[0].col_ptr.numel())
            self.row_ptr = _assemble(dev, torch.int64, batch * rows + 1, [
                (s.row_ptr, b * rows, rows + (1 if b == batch - 1 else 0), e[b])
                for b, s in enumerate(structs)])
            self.col_ptr = _assemble(dev, torch.int64, batch * (lp - 1) + 1, [
                (s.col_ptr, b * (lp - 1), lp - (0 if b == batch - 1 else 1), e[b])
                for b, s in enumerate(structs)])
            if self.nnz:
                self.cols = _assemble(dev, torch.int32, self.nnz, [
                    (s.cols0, e[b], s.nnz, b * slot_stride) for b, s in enumerate(structs)])
                self.col_ent = _assemble(dev, torch.int64, self.nnz, [
                    (s.col_ent, e[b], s.nnz, e[b]) for b, s in enumerate(structs)])
                self.col_row = _assemble(dev, torch.int32, self.nnz, [
                    (s.col_row, e[b], s.nnz, b * rows) for b, s in enumerate(structs)])
            else:
                self.cols = torch.zeros(1, dtype=torch.int32, device=dev)
                self.col_ent = torch.zeros(1, dtype=torch.int64, device=dev)
                self.col_row = torch.zeros(1, dtype=torch.int32, device=dev)
            # hub rows of every slot first, then the remaining rows of every slot
            if rows:
                hubs = np.cumsum([0] + [s.n_hub for s in structs])
                rest = np.cumsum([0] + [rows - s.n_hub for s in structs])
                segs = [(s.order, int(hubs[b]), s.n_hub, b * rows)
                        for b, s in enumerate(structs)]
                segs += [(s.order, int(hubs[-1] + rest[b]), rows - s.n_hub, b * rows, s.n_hub)
                         for b, s in enumerate(structs)]
                self.order = _assemble(dev, torch.int32, batch * rows, segs)
            else:
                self.order = torch.zeros(1, dtype=torch.int32, device=dev)
        self.n_hub = sum(s.n_hub for s in structs)
        nr = max(batch * rows, 1)
        # every row's rdeg / sol / cand and the residual counts are written by
        # s2v_shard_init (no fill launches)
        alloc = torch.empty if rows else torch.zeros
        self.rdeg = alloc(nr, dtype=torch.int32, device=dev)
        self.sol_d = alloc(nr, dtype=torch.uint8, device=dev)
        self.cand_d = alloc(nr, dtype=torch.uint8, device=dev)
        self.residual_d = torch.empty(batch, dtype=torch.int64, device=dev)
        self._shard = _lib.s2v_shard(
            num_nodes=n, batch=batch, world=P, rank=part.rank, _pad=0,
            row_start=part.row_start, num_rows=rows, rows_max=self.rows_max, nnz=self.nnz,
            row_ptr=ptr(self.row_ptr), cols=ptr(self.cols), col_ptr=ptr(self.col_ptr),
            col_ent=ptr(self.col_ent), col_row=ptr(self.col_row), rdeg=ptr(self.rdeg),
            sol=ptr(self.sol_d), cand=ptr(self.cand_d), residual=ptr(self.residual_d),
            order=ptr(self.order), n_hub=self.n_hub)
        if P == 1:  # the physical layout is the node layout
            sol_phys = np.ascontiguousarray(solutions)
        else:
            sol_phys = np.zeros((batch, P, self.rows_max), dtype=np.uint8)
            for r, pr in enumerate(partition_rows(n, P)):
                sol_phys[:, r, :pr.num_rows] = solutions[:, pr.row_start:pr.row_stop]
        sol_phys_d = to_device(sol_phys.reshape(-1), dev, pinned=True)
        _lib.call("s2v_shard_init", ctypes.byref(self._shard), ptr(cols_src), ptr(sol_phys_d),
                  stream_ptr())
        self._host = {}
        self._ws: dict = {}

    # -- C view ------------------------------------------------------------

    @property
    def shard(self) -> ctypes.Structure:
        return self._shard

    def shard_ref(self):
        return ctypes.byref(self._shard)

    colsum_cache = None

    @contextlib.contextmanager
    def active_rows(self, rows: torch.Tensor, count: torch.Tensor, colsum_cache=None,
                    csr=None, sol_all=None):
        """Within the block, forward rounds and the scorer visit only the rows
        of the active list `rows` (int32, count[0] entries, count[1] hub rows
        first; s2v_active_compact) -- the residual rows of an episode.
        colsum_cache: the caller's dict for the incremental global sum
        (s2v_colsum_residual with `last`), valid for fixed parameters.
        csr: (row_ptr, cols) compact CSR of the list (s2v_active_compact).
        sol_all: P > 1 with csr -- S of every physical row (s2v_sol_mark)."""
        sh = self._shard
        sh.active, sh.active_n = ptr(rows), ptr(count)
        if csr is not None:
            sh.active_ptr, sh.active_cols = ptr(csr[0]), ptr(csr[1])
            if sol_all is not None:
                sh.active_sol = ptr(sol_all)
        self.colsum_cache = colsum_cache
        try:
            yield
        finally:
            sh.active, sh.active_n, sh.active_ptr, sh.active_cols = None, None, None, None
            sh.active_sol = None
            self.colsum_cache = None

    @property
    def active_on(self) -> bool:
        return bool(self._shard.active)

    def workspace(self, name: str, key, make):
        """Per-state cache of device scratch buffers (reused across steps)."""
        entry = self._ws.get(name)
        if entry is None or entry[0] != key:
            entry = (key, make())
            self._ws[name] = entry
        return entry[1]

    def invalidate(self) -> None:
        self._host.clear()

    def release(self) -> None:
        """Drop this state's device workspaces now (embedding buffers, score
        and backward scratch): a caller replacing states in a loop returns
        their memory to the caching allocator at once instead of at the
        next cycle collection.  The state stays usable (workspaces are
        rebuilt on demand)."""
        self._ws.clear()
        self._host.clear()

    def _mirror(self, name: str, tensor: torch.Tensor, shape) -> np.ndarray:
        arr = self._host.get(name)
        if arr is None:
            arr = tensor.to("cpu").numpy()[:int(np.prod(shape))].reshape(shape)
            self._host[name] = arr
        return arr

    # -- views (state.py:140-155) -------------------------------------------

    @property
    def sol(self) -> np.ndarray:
        return self._mirror("sol", self.sol_d, (self.batch, self.part.num_rows))

    @property
    def cand(self) -> np.ndarray:
        return self._mirror("cand", self.cand_d, (self.batch, self.part.num_rows))

    @property
    def local_residual(self) -> np.ndarray:
        return self._mirror("residual", self.residual_d, (self.batch,))

    def local_degrees(self) -> np.ndarray:
        """(B, rows) residual degree of each locally owned node."""
        deg = self._mirror("rdeg", self.rdeg, (self.batch, self.part.num_rows))
        return deg.astype(self.dtype)

    def local_residual_coo(self, slot: int) -> tuple[np.ndarray, np.ndarray]:
        """Surviving (global row, col) entries of one graph's local slice."""
        rows = self.part.num_rows
        rp = self.row_ptr.to("cpu").numpy()
        lo, hi = int(rp[slot * rows]), int(rp[(slot + 1) * rows])
        cols = (self.cols[lo:hi].to("cpu").numpy().view(np.uint32) if hi > lo
                else np.zeros(0, np.uint32))
        alive = (cols & np.uint32(0x80000000)) == 0
        phys = (cols & np.uint32(0x7FFFFFFF)).astype(np.int64)
        local_rows = np.repeat(np.arange(rows), np.diff(rp[slot * rows:(slot + 1) * rows + 1]))
        inv = np.empty(self.world * self.rows_max, dtype=np.int64)
        inv.fill(-1)
        inv[phys_rows(self.num_nodes, self.world)] = np.arange(self.num_nodes)
        slot_phys = phys - slot * self.world * self.rows_max
        return (local_rows[alive] + self.part.row_start, inv[slot_phys[alive]])

    # -- mutation (state.py:173-208) -------------------------------------------

    def apply_action(self, v: int, slot: int = 0) -> None:
        """Move node v into the partial solution of one batched graph.
        Validation is owner-side, with the reference's messages."""
        if not 0 <= v < self.num_nodes:
            raise InvalidActionError(f"node {v} out of range [0, {self.num_nodes})")
        if not 0 <= slot < self.batch:
            raise InvalidActionError(f"batch slot {slot} out of range")
        if self.part.owns(v):
            i = v - self.part.row_start
            if self.sol[slot, i]:
                raise InvalidActionError(f"node {v} is already in the solution")
            if not self.cand[slot, i]:
                raise InvalidActionError(f"node {v} is not a candidate")
        picks = np.full((self.batch, 1), -1, dtype=np.int64)
        picks[slot, 0] = v
        self.apply_groups(picks, comm=None)

    def apply_groups(self, picks: np.ndarray, comm=None):
        """Apply a group of picks per slot with the mid-group skip rule
        (inference.py:125-146).  picks: (B, d) int64, -1 padded.  Returns
        (applied (B, d) bool, removed (B,) global entries removed).  Groups
        wider than 64 run as consecutive sub-groups of 64; only the group's
        first pick is applied unconditionally, as in the reference."""
        picks = np.ascontiguousarray(picks, dtype=np.int64)
        B, d = picks.shape
        if d > 64:
            parts = [self._apply_chunk(np.ascontiguousarray(picks[:, c:c + 64]), comm, c == 0)
                     for c in range(0, d, 64)]
            return (np.concatenate([a for a, _ in parts], axis=1),
                    np.sum([r for _, r in parts], axis=0))
        return self._apply_chunk(picks, comm, True)

    def _apply_chunk(self, picks: np.ndarray, comm, first_forced: bool):
        B, d = picks.shape
        ws = self.workspace("apply", d, lambda: {
            "picks": torch.empty(B * d, dtype=torch.int64, device=self.device),
            "info": torch.empty(2 * B * d, dtype=torch.int64, device=self.device),
            # one read-back: [removed B | residual B | applied B*d bytes]
            "out": torch.empty(2 * B + (B * d + 7) // 8, dtype=torch.int64, device=self.device)})
        ws["picks"].copy_(torch.from_numpy(picks.reshape(-1)), non_blocking=False)
        st = stream_ptr()
        _lib.call("s2v_apply_phase1", self.shard_ref(), ptr(ws["picks"]), d, ptr(ws["info"]), 0,
                  None, st)
        if self.world > 1 and (d > 1 or not first_forced):
            dc = comm.device_comm() if comm is not None else None
            if dc is None:
                raise InvalidActionError("a sharded state needs its comm to apply picks")
            dc.allreduce(ptr(ws["info"]), ws["info"].numel(), 0, st)
        out = ws["out"]
        base = out.data_ptr()
        _lib.call("s2v_apply_phase2", self.shard_ref(), ptr(ws["picks"]), d, ptr(ws["info"]),
                  base + 16 * B, base, 1 if first_forced else 0, st)
        _lib.call("s2v_memcpy_async", base + 8 * B, ptr(self.residual_d), 8 * B, st)
        self.invalidate()
        host = out.to("cpu").numpy()
        removed = host[:B].copy()
        self._host["residual"] = host[B:2 * B].copy()
        applied = host[2 * B:].view(np.uint8)[:B * d].reshape(B, d).astype(bool)
        return applied, removed

    # -- termination (state.py:212-220) ------------------------------------------

    def residual_counts(self, comm) -> np.ndarray:
        """(B,) global residual adjacency entry counts (sum-all-reduce)."""
        return comm.all_reduce_sum(self.local_residual, tag="env")

    def is_covered(self, slot: int, comm) -> bool:
        if not 0 <= slot < self.batch:
            raise InvalidActionError(f"batch slot {slot} out of range")
        return int(self.residual_counts(comm)[slot]) == 0


def apply_action(state: PartitionedState, v: int, slot: int = 0) -> PartitionedState:
    state.apply_action(v, slot)
    return state


def is_covered(state: PartitionedState, slot: int, comm) -> bool:
    return state.is_covered(slot, comm)
