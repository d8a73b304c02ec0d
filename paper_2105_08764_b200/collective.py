"""Worker groups: host rendezvous collectives + NCCL device collectives.

API mirrors pkg/src/graphrl/collective.py (WorkerGroup, Comm, run_workers,
CollectiveStats).  Two kinds of traffic:

* host collectives on small numpy arrays (candidacy flags, targets, counts):
  rank-ordered, by value, exactly the reference semantics -- through an
  in-process rendezvous when ranks are threads (run_workers), or through
  torch.distributed (gloo) when ranks are processes (torchrun, DistComm);
* device collectives on HBM buffers (per-round halo all-gather of embeddings,
  selection info, gradient packs): NCCL over NVLink, owned by libs2v
  (s2v_comm_*), one communicator per rank, created lazily.

Each rank binds one CUDA device: rank r of a thread group uses device
r % device_count, a torchrun process uses LOCAL_RANK.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np

from .errors import CollectiveAborted, CollectiveError

DEFAULT_TIMEOUT = 30.0


@dataclass
class CollectiveStats:
    """Per-tag instrumentation: logical calls and per-rank elements sent."""
    calls: int = 0
    elements: int = 0


class WorkerGroup:
    """A fixed set of P cooperating thread-ranks and their rendezvous."""

    def __init__(self, num_workers: int, timeout: float = DEFAULT_TIMEOUT,
                 use_nccl: bool = False):
        if num_workers < 1:
            raise ValueError(f"num_workers must be >= 1, got {num_workers}")
        self.num_workers = int(num_workers)
        self.timeout = float(timeout)
        self._slots: list = [None] * self.num_workers
        self._barrier = threading.Barrier(self.num_workers)
        self._stats: dict[str, CollectiveStats] = {}
        self._lock = threading.Lock()
        self.use_nccl = bool(use_nccl)

    def comm(self, rank: int) -> "Comm":
        if not 0 <= rank < self.num_workers:
            raise ValueError(f"rank {rank} out of range for P={self.num_workers}")
        return Comm(self, rank)

    def abort(self) -> None:
        self._barrier.abort()

    def stats_snapshot(self) -> dict[str, CollectiveStats]:
        with self._lock:
            return {t: CollectiveStats(s.calls, s.elements) for t, s in self._stats.items()}

    def reset_stats(self) -> None:
        with self._lock:
            self._stats.clear()

    def _record(self, tag: str, elements: int) -> None:
        with self._lock:
            st = self._stats.setdefault(tag, CollectiveStats())
            st.calls += 1
            st.elements += int(elements)

    def _wait(self) -> None:
        try:
            self._barrier.wait(timeout=self.timeout)
        except threading.BrokenBarrierError:
            raise CollectiveAborted(
                f"collective aborted: a rank failed or did not arrive within "
                f"{self.timeout:.1f}s (P={self.num_workers})") from None

    def _exchange_objects(self, rank: int, value) -> list:
        """Rank-ordered exchange of arbitrary Python objects (no copy)."""
        self._slots[rank] = value
        self._wait()
        out = list(self._slots)
        self._wait()
        return out

    def _exchange(self, rank: int, value) -> list:
        # deposit a private copy, wait for everyone, snapshot, wait again so
        # no rank overwrites its slot before all peers have read it
        self._slots[rank] = np.array(value, copy=True)
        self._wait()
        out = list(self._slots)
        self._wait()
        return out


class _DeviceComm:
    """NCCL communicator of one rank (libs2v s2v_comm_*)."""

    def __init__(self, unique_id: bytes, world: int, rank: int):
        from . import _lib
        self._lib = _lib
        handle = ctypes.c_void_p()
        buf = ctypes.create_string_buffer(unique_id, len(unique_id))
        _lib.call("s2v_comm_init", buf, world, rank, ctypes.byref(handle))
        self.handle = handle
        self.world, self.rank = world, rank
        self._scratch: dict = {}  # all-gather scratch of the ordered all-reduce, by bytes

    supports_push = False

    def allgather_rows(self, tensor, chunk_bytes: int, slot_stride: int, nslots: int,
                       stream: int, peers=None) -> None:
        self._lib.call("s2v_comm_allgather_slots", self.handle, tensor.data_ptr(), chunk_bytes,
                       slot_stride, nslots, self.rank, stream)

    def allreduce(self, buf_ptr: int, count: int, kind: int, stream: int) -> None:
        """Rank-ordered sum (all-gather + s2v_sum_ranks_typed), not
        ncclAllReduce: the reference adds rank 0, 1, ... in order
        (collective.py:114-116) and NCCL's ring order is not that."""
        import torch
        if count == 0:
            return
        nbytes = count * (4 if kind == 2 else 8)
        buf = self._scratch.get(nbytes)
        if buf is None:
            buf = self._scratch[nbytes] = torch.empty(self.world * nbytes, dtype=torch.uint8,
                                                      device="cuda")
        self._lib.call("s2v_comm_allreduce_ordered", self.handle, buf_ptr, count, kind,
                       buf.data_ptr(), stream)

    def close(self) -> None:
        if self.handle:
            self._lib.load().s2v_comm_destroy(self.handle)
            self.handle = None


class _PeerTransport:
    """Peer-memory device transport (NVLink P2P loads/stores between ranks).

    Every rank maps its peers' same-role buffers (peers_of: a collective
    registration, cached per workspace by the callers); the forward round
    kernel pushes each output row into every peer's halo buffer itself
    (s2v_embed_round_peers -- the exchange is fused into the compute), and
    ranks order producer/consumer on the CUDA streams: per-peer flags written
    and waited on by the streams for process ranks, CUDA events for thread
    ranks (no host synchronisation of GPU work, no SM spinning).  All-reduces push each rank's vector into every peer's
    scratch row [rank] and sum the P rows in ascending rank order on the
    device (s2v_sum_ranks_typed): the reference's order
    (collective.py:100-117), identical bits on every rank.
    Subclasses supply peers_of (thread-ranks: plain addresses exchanged
    through the host rendezvous; process ranks: CUDA IPC handles).
    """

    supports_push = True

    def _init_flags(self):
        import torch
        self.epoch = 0
        self.flags = torch.zeros(max(self.world, 1) * 8, dtype=torch.int32, device="cuda")
        self.peer_flags = self.peers_of(self.flags)
        self._scratch: dict = {}

    def peers_of(self, tensor) -> list[int]:  # pragma: no cover - abstract
        raise NotImplementedError

    def peer_array(self, tensor):
        """peers_of as a device array of pointers (kernel argument)."""
        import torch
        return torch.tensor(self.peers_of(tensor), dtype=torch.int64, device=tensor.device)

    def signal_and_wait(self, stream: int) -> None:
        """Stream-ordered all-rank barrier: after this rank's prior work, raise
        its flag in every peer; before later work, wait for every peer's."""
        self.epoch += 1
        for q in range(self.world):
            self._lib.call("s2v_stream_write_u32", self.peer_flags[q] + 4 * self.rank,
                           self.epoch, stream)
        own = self.flags.data_ptr()
        for q in range(self.world):
            self._lib.call("s2v_stream_wait_u32", own + 4 * q, self.epoch, stream)

    def allgather_rows(self, tensor, chunk_bytes: int, slot_stride: int, nslots: int,
                       stream: int, peers=None) -> None:
        """Pull every peer's chunk of each slot (generic layouts; the K = 64
        rounds push instead)."""
        if peers is None:
            peers = self.peers_of(tensor)
        self.signal_and_wait(stream)  # every producer is done
        own = tensor.data_ptr()
        for q in range(self.world):
            if q == self.rank:
                continue
            for b in range(nslots):
                off = b * slot_stride + q * chunk_bytes
                self._lib.call("s2v_memcpy_async", own + off, peers[q] + off, chunk_bytes, stream)
        self.signal_and_wait(stream)  # every reader is done before buffers are reused

    def allreduce(self, buf_ptr: int, count: int, kind: int, stream: int) -> None:
        """In-place ascending-rank sum of count elements (kind 0 int64,
        1 fp64, 2 fp32) across the ranks, entirely on the device.  Two scratch
        buffers per (count, kind) alternate: the signal of the next
        all-reduce separates a reuse from every peer's read of it."""
        import torch
        if count == 0:
            return
        item = 4 if kind == 2 else 8
        nbytes = count * item
        ent = self._scratch.get((count, kind))
        if ent is None:
            bufs = [torch.empty(self.world * nbytes, dtype=torch.uint8, device="cuda")
                    for _ in range(2)]
            ent = self._scratch[(count, kind)] = [bufs, [self.peers_of(b) for b in bufs], 0]
        bufs, peers, par = ent
        ent[2] ^= 1
        for q in range(self.world):
            self._lib.call("s2v_memcpy_async", peers[par][q] + self.rank * nbytes, buf_ptr,
                           nbytes, stream)
        self.signal_and_wait(stream)  # every rank's row has landed
        self._lib.call("s2v_sum_ranks_typed", kind, self.world, count, bufs[par].data_ptr(),
                       buf_ptr, stream)


class _LocalDeviceComm(_PeerTransport):
    """Peer-memory transport for thread-ranks of one process (run_workers).

    Ranks may share one GPU (tests on a single B200) or own one each (peer
    access enabled between every pair of the group's devices).  Every rank
    runs on its own CUDA stream (run_workers), so one rank's stream waiting
    on a flag never blocks a peer sharing the device."""

    def __init__(self, comm: "Comm"):
        import torch
        from . import _lib
        self._lib = _lib
        self.comm = comm
        self.world, self.rank = comm.size, comm.rank
        dev = torch.cuda.current_device()
        for other in self._publish(dev):
            _lib.call("s2v_enable_peer_access", int(other))
        self._init_flags()

    def _publish(self, value):
        return self.comm.group._exchange_objects(self.rank, value)

    def _init_flags(self):
        self.epoch = 0
        self._scratch: dict = {}

    def signal_and_wait(self, stream: int) -> None:
        """Stream-ordered all-rank barrier with CUDA events: each rank records
        an event after its prior work and its stream waits on every peer's.
        (Stream waits on peer-written flags can deadlock when thread-ranks
        share a device: their streams may share a hardware queue.)  The host
        threads only exchange the event handles; no GPU work is waited on."""
        import torch
        ev = torch.cuda.Event()
        ev.record(torch.cuda.ExternalStream(stream))
        for q, peer_ev in enumerate(self._publish(ev)):
            if q != self.rank:
                torch.cuda.ExternalStream(stream).wait_event(peer_ev)

    def peers_of(self, tensor) -> list[int]:
        """Every rank's address of the same-role buffer (own included);
        collective, same contract as the IPC transport's."""
        return [int(p) for p in self._publish(tensor.data_ptr())]

    def close(self) -> None:
        pass


class _IpcDeviceComm(_PeerTransport):
    """Peer-memory transport for process ranks (torchrun / DistComm): peer
    buffers mapped with CUDA IPC.  Ranks may share a GPU (tests) or own one
    each (NVLink P2P)."""

    def __init__(self, comm: "DistComm"):
        from . import _lib
        self._lib = _lib
        self.comm = comm
        self.world, self.rank = comm.size, comm.rank
        self._imports: dict[bytes, int] = {}
        self._init_flags()

    def _export(self, ptr: int):
        handle = ctypes.create_string_buffer(64)
        off = ctypes.c_uint64()
        self._lib.call("s2v_ipc_export", ptr, handle, ctypes.byref(off))
        return handle.raw, int(off.value)

    def _import(self, handle: bytes) -> int:
        base = self._imports.get(handle)
        if base is None:
            out = ctypes.c_void_p()
            self._lib.call("s2v_ipc_import", ctypes.create_string_buffer(handle, 64),
                           ctypes.byref(out))
            base = int(out.value)
            self._imports[handle] = base
        return base

    def peers_of(self, tensor) -> list[int]:
        """Every rank's address of the same-role buffer (own included).

        Collective: every rank must register its same-role buffer at the same
        point (callers cache the result per workspace, never by address --
        allocator address reuse differs across ranks)."""
        handle, off = self._export(tensor.data_ptr())
        allh = self.comm._gather_objects((handle, off))
        return [tensor.data_ptr() if q == self.rank else self._import(h) + o
                for q, (h, o) in enumerate(allh)]

    def close(self) -> None:
        for base in self._imports.values():
            self._lib.load().s2v_ipc_close(base)
        self._imports.clear()


def _new_unique_id() -> bytes:
    from . import _lib
    buf = ctypes.create_string_buffer(128)
    _lib.call("s2v_comm_unique_id", buf, 128)
    return buf.raw


class Comm:
    """Per-rank handle used to enter collectives (collective.py:92-146)."""

    def __init__(self, group: WorkerGroup, rank: int):
        self.group = group
        self.rank = rank
        self.size = group.num_workers
        self._dev = None

    # -- host collectives (reference semantics) -----------------------------

    def all_reduce_sum(self, local, tag: str = "default") -> np.ndarray:
        arr = np.asarray(local)
        if self.rank == 0:
            self.group._record(tag, arr.size)
        slots = self.group._exchange(self.rank, arr)
        shapes = [s.shape for s in slots]
        if any(s != shapes[0] for s in shapes):
            raise CollectiveError(f"all_reduce_sum shape mismatch across ranks: {shapes}")
        out = slots[0].astype(np.result_type(*[s.dtype for s in slots]), copy=True)
        for other in slots[1:]:
            out += other
        return out

    def all_gather(self, local, axis: int = -1, tag: str = "default") -> np.ndarray:
        arr = np.asarray(local)
        if self.rank == 0:
            self.group._record(tag, arr.size)
        slots = self.group._exchange(self.rank, arr)
        ref = list(slots[0].shape)
        ax = axis % max(slots[0].ndim, 1) if slots[0].ndim else 0
        for s in slots:
            shp = list(s.shape)
            if len(shp) != len(ref):
                raise CollectiveError(f"all_gather rank mismatch: {[t.shape for t in slots]}")
            if shp[:ax] != ref[:ax] or shp[ax + 1:] != ref[ax + 1:]:
                raise CollectiveError(
                    f"all_gather shape mismatch off the concat axis: {[t.shape for t in slots]}")
        if self.size == 1:
            return slots[0].copy()
        return np.concatenate(slots, axis=axis)

    def barrier(self) -> None:
        self.group._wait()

    # -- device collectives ------------------------------------------------

    def record(self, tag: str, elements: int) -> None:
        if self.rank == 0:
            self.group._record(tag, elements)

    def device_comm(self):
        """This rank's device transport (None when P == 1): peer copies between
        the thread-ranks of this process (_LocalDeviceComm), or NCCL when the
        group was created with use_nccl=True and every rank owns a GPU."""
        if self.size == 1:
            return None
        if self._dev is None:
            if getattr(self.group, "use_nccl", False):
                uid = _new_unique_id() if self.rank == 0 else b""
                ids = self.group._exchange(self.rank, np.frombuffer(uid or b"\0", dtype=np.uint8))
                self._dev = _DeviceComm(bytes(ids[0]), self.size, self.rank)
            else:
                self._dev = _LocalDeviceComm(self)
        return self._dev


class DistComm:
    """Comm over torch.distributed for one-process-per-GPU runs (torchrun).

    Host collectives go through a gloo group (CPU numpy payloads); device
    collectives through libs2v's own NCCL communicator.
    """

    def __init__(self):
        import torch.distributed as dist
        if not dist.is_initialized():
            raise RuntimeError("DistComm needs torch.distributed to be initialised")
        self._dist = dist
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()
        self._gloo = dist.new_group(backend="gloo")
        self._stats: dict[str, CollectiveStats] = {}
        self.group = self
        self._dev = None

    def stats_snapshot(self):
        return dict(self._stats)

    def record(self, tag: str, elements: int) -> None:
        if self.rank == 0:
            st = self._stats.setdefault(tag, CollectiveStats())
            st.calls += 1
            st.elements += int(elements)

    def _gather_objects(self, arr):
        out = [None] * self.size
        self._dist.all_gather_object(out, arr, group=self._gloo)
        return out

    def all_reduce_sum(self, local, tag: str = "default") -> np.ndarray:
        arr = np.asarray(local)
        self.record(tag, arr.size)
        slots = self._gather_objects(arr)
        out = slots[0].astype(np.result_type(*[s.dtype for s in slots]), copy=True)
        for other in slots[1:]:
            out += other
        return out

    def all_gather(self, local, axis: int = -1, tag: str = "default") -> np.ndarray:
        arr = np.asarray(local)
        self.record(tag, arr.size)
        slots = self._gather_objects(arr)
        return slots[0].copy() if self.size == 1 else np.concatenate(slots, axis=axis)

    def barrier(self) -> None:
        self._dist.barrier(group=self._gloo)

    def device_comm(self):
        """IPC peer-memory transport (fused halo exchange) by default;
        S2V_TRANSPORT=nccl selects NCCL collectives instead."""
        if self.size == 1:
            return None
        if self._dev is None:
            if os.environ.get("S2V_TRANSPORT", "ipc") == "nccl":
                uid = [_new_unique_id() if self.rank == 0 else None]
                self._dist.broadcast_object_list(uid, src=0, group=self._gloo)
                self._dev = _DeviceComm(uid[0], self.size, self.rank)
            else:
                self._dev = _IpcDeviceComm(self)
        return self._dev


def run_workers(num_workers: int, fn, *args, timeout: float = DEFAULT_TIMEOUT,
                group: WorkerGroup | None = None, bind_devices: bool = True) -> list:
    """Run fn(comm, *args) on every rank (one thread per rank, each bound to
    one CUDA device); results in rank order.  The first failure aborts the
    group and is re-raised, root causes before knock-on aborts
    (collective.py:149-195)."""
    if group is None:
        group = WorkerGroup(num_workers, timeout=timeout)
    elif group.num_workers != num_workers:
        raise ValueError("group size does not match num_workers")

    def bind(rank: int) -> None:
        if not bind_devices:
            return
        import torch
        if torch.cuda.is_available():
            from .device import bind_device
            bind_device(rank % torch.cuda.device_count())

    if num_workers == 1:
        bind(0)
        return [fn(group.comm(0), *args)]

    results: list = [None] * num_workers
    failures: list[tuple[int, BaseException]] = []
    lock = threading.Lock()

    def runner(rank: int) -> None:
        try:
            bind(rank)
            stream = None
            if bind_devices:
                import torch
                if torch.cuda.is_available():
                    # one stream per rank: the device transports order ranks
                    # with stream waits on flags, which must never block a
                    # peer rank sharing the device
                    stream = torch.cuda.Stream()
            if stream is None:
                results[rank] = fn(group.comm(rank), *args)
            else:
                import torch
                with torch.cuda.stream(stream):
                    results[rank] = fn(group.comm(rank), *args)
                stream.synchronize()
        except BaseException as exc:  # noqa: BLE001 -- re-raised below
            with lock:
                failures.append((rank, exc))
            group.abort()

    threads = [threading.Thread(target=runner, args=(r,), name=f"s2v-rank-{r}")
               for r in range(num_workers)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if failures:
        def precedence(item):
            exc = item[1]
            if isinstance(exc, CollectiveAborted):
                return 2
            if isinstance(exc, CollectiveError):
                return 1
            return 0
        failures.sort(key=lambda it: (precedence(it), it[0]))
        raise failures[0][1]
    return results


def local_rank_from_env() -> int:
    return int(os.environ.get("LOCAL_RANK", "0"))
