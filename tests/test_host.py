"""CPU: host-side pieces of the API (no device work) and the N > 1 host
protocol over torch.distributed/gloo with world_size 2."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2105_08764_b200 as P
from paper_2105_08764_b200.policy import decode_keys, merge_rank_keys


class TestSelection:
    """pkg/tests/test_inference.py:13-60."""

    def test_default_ladder(self):
        s = P.SelectionSchedule.adaptive()
        assert [s.d_for(c, 1000) for c in (501, 500, 251, 250, 126, 125, 1)] == \
            [8, 4, 4, 2, 2, 1, 1]

    def test_validation(self):
        with pytest.raises(ValueError, match="decreasing"):
            P.SelectionSchedule(thresholds=((0.25, 4), (0.5, 8)))
        with pytest.raises(ValueError, match="non-increasing"):
            P.SelectionSchedule(thresholds=((0.5, 2), (0.25, 4)))
        with pytest.raises(ValueError, match=">= 1"):
            P.SelectionSchedule(thresholds=((0.5, 0),))

    def test_top_d(self):
        assert P.select_top_d(np.array([5.0, 1, 9, 9]), np.array([1, 0, 1, 1], bool), 2) == [2, 3]
        assert P.select_top_d(np.array([3.0, 2, 1, 0]), np.array([1, 1, 0, 1], bool), 10) == \
            [0, 1, 3]
        with pytest.raises(P.InvalidActionError, match="empty"):
            P.select_top_d(np.zeros(3), np.zeros(3, bool), 1)


class TestPartitionAndReplay:
    def test_partition_rows(self):
        assert [(p.row_start, p.row_stop) for p in P.partition_rows(7, 2)] == [(0, 4), (4, 7)]
        with pytest.raises(ValueError):
            P.partition_rows(3, 4)

    def test_pack_roundtrip_and_fifo(self):
        bits = (np.random.default_rng(0).random(37) < 0.5).astype(np.uint8)
        assert np.array_equal(P.unpack_solution(P.pack_solution(bits), 37), bits)
        buf = P.ReplayBuffer(3)
        for i in range(5):
            buf.add(P.ExperienceTuple(i, b"", 0, 0.0))
        assert [buf[i].graph_index for i in range(3)] == [2, 3, 4]
        with pytest.raises(ValueError):
            P.ExperienceTuple(0, b"", 0, float("nan"))

    def test_epsilon(self):
        cfg = P.TrainConfig(eps_start=0.9, eps_end=0.1, eps_decay_steps=500)
        assert cfg.epsilon_at(0) == 0.9 and cfg.epsilon_at(10_000) == pytest.approx(0.1)


class TestCheckpoint:
    """pkg/tests/test_policy.py:384-407: GRLP format unchanged."""

    def test_roundtrip_and_errors(self, tmp_path):
        params = P.PolicyParams.initialize(32, 2, seed=4)
        path = tmp_path / "c.bin"
        P.save_checkpoint(params, path)
        back = P.load_checkpoint(path)
        assert back.num_layers == 2 and back.dtype == np.float32
        for n in P.PARAM_NAMES:
            assert getattr(back, n).tobytes() == getattr(params, n).tobytes()
        (tmp_path / "bad.bin").write_bytes(b"NOPE" + b"\0" * 32)
        with pytest.raises(P.DataError, match="magic"):
            P.load_checkpoint(tmp_path / "bad.bin")


class TestHostCollectives:
    def test_thread_group_semantics(self):
        group = P.WorkerGroup(3)

        def worker(comm):
            s = comm.all_reduce_sum(np.array([comm.rank + 1.0]), tag="t")
            g = comm.all_gather(np.array([comm.rank]), axis=-1)
            return s, g
        outs = P.run_workers(3, worker, group=group, bind_devices=False)
        for s, g in outs:
            assert s.tolist() == [6.0] and g.tolist() == [0, 1, 2]
        assert group.stats_snapshot()["t"].calls == 1

    def test_failure_propagates(self):
        def worker(comm):
            if comm.rank == 1:
                raise RuntimeError("boom")
            comm.barrier()
        with pytest.raises(RuntimeError, match="boom"):
            P.run_workers(2, worker, timeout=2.0, bind_devices=False)


def _keys(scores, nodes):
    """Host restatement of the device key image (s2v_common.cuh make_key)."""
    out = np.zeros((len(scores), 2), np.uint64)
    for i, (s, v) in enumerate(zip(scores, nodes)):
        b = np.array([s], np.float64).view(np.uint64)[0]
        if s == 0:
            b = np.uint64(0)
        sign = np.uint64(1) << np.uint64(63)
        out[i, 0] = ~b if (b & sign) else (b | sign)
        out[i, 1] = ~np.uint64(v)
    return out


def test_key_image_round_trips_and_orders():
    scores = np.array([1.5, -2.0, 0.0, -0.0, 3.25, 1.5], np.float32)
    nodes = np.arange(6)
    k = _keys(scores.astype(np.float64), nodes)
    n, v, ok = decode_keys(k)
    assert np.array_equal(n, nodes) and ok.all()
    assert np.array_equal(v.astype(np.float32), np.where(scores == 0, 0, scores))
    order = np.lexsort((k[:, 1], k[:, 0]))[::-1]
    # descending score, ties -> lowest node, -0 == +0
    assert order.tolist() == [4, 0, 5, 2, 3, 1]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = P.DistComm()
        total = comm.all_reduce_sum(np.array([rank + 1, 10 * rank], np.int64))
        gathered = comm.all_gather(np.array([rank, rank]), axis=-1)
        # per-rank top-2 keys of a row-partitioned score vector, merged
        scores = np.array([0.5, 2.0, 2.0, -1.0, 7.0, 2.0], np.float64)
        lo, hi = (0, 3) if rank == 0 else (3, 6)
        loc = scores[lo:hi]
        order = np.lexsort((-np.arange(lo, hi), loc))[::-1][:2]
        top = _keys(loc[order], np.arange(lo, hi)[order])[None]
        merged, counts = merge_rank_keys(top, np.array([3]), comm, 3)
        nodes, vals, _ = decode_keys(merged)
        q.put((rank, total.tolist(), gathered.tolist(), nodes[0].tolist(), counts.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_host_protocol():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, total, gathered, nodes, counts in res:
        assert total == [3, 10]
        assert gathered == [0, 0, 1, 1]
        # global top-3 of [0.5, 2, 2, -1, 7, 2]: 7 (node 4), then the 2.0 tie
        # broken by lowest index: nodes 1, 2
        assert nodes == [4, 1, 2]
        assert counts == [6]


def test_bench_peak_parser(tmp_path, monkeypatch):
    """bench.py's roofline peak: a sustained HBM figure from the
    driver-written MEASURED_PEAKS.json when present (GB/s or TB/s), else the
    profiling recipe's fallback."""
    import bench
    f = tmp_path / "MEASURED_PEAKS.json"
    monkeypatch.setattr(bench, "MEASURED", f)
    assert bench.peaks()[0] == 6650.0
    f.write_text('{"hbm": {"burst_gbs": 7400, "sustained_gbs": 6900}, "bf16_tflops": 2200}')
    assert bench.peaks()[0] == 6900.0
    f.write_text('{"copy_bandwidth_tbs": 6.8}')
    assert bench.peaks()[0] == 6800.0
    f.write_text('{"bf16_tflops": 2200}')
    assert bench.peaks()[0] == 6650.0
