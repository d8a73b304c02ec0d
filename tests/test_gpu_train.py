"""Training path on the GPU vs the reference: golden losses/grads/params of a
reference training step (tests/golden/train_*.npz) and the numpy port
(oracle/port.py) on random cases; tolerance 1e-4 relative,
Adam bitwise."""
from pathlib import Path

import numpy as np
import pytest

import paper_2105_08764_b200 as P
from oracle import port
from reference_math import scale_error

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("name,tol", [("train_ba1000_b4_k64_l5", 1e-4),
                                      ("train_ba600_b3_k16_l3_f64", 1e-9),
                                      ("train_cfg2_ba10k_b32_k64_l5", 1e-4)])
def test_training_step_matches_reference(name, tol):
    """Reference training steps (oracle/make_golden.py).  train_cfg2_* is
    BASELINE configs[1] itself: 32 x BA(10000,4,100+i), B = 32, tau = 4; at
    B = 32 the Bellman targets go through the device u1's sequential-sgemm
    branch (csrc/s2v_episode.cu), which they pin bitwise."""
    path = GOLD / f"{name}.npz"
    if not path.exists():
        pytest.skip("golden fixture not generated")
    z = np.load(path)
    n, m, B, K, L, tau = (int(z[k]) for k in ("n", "m", "B", "K", "L", "tau"))
    dtype = z["p0_theta1"].dtype
    dataset = [P.generate_ba(n, m, 100 + i) for i in range(B)]
    params = P.PolicyParams(num_layers=L, **{k: z[f"p0_{k}"].copy() for k in P.PARAM_NAMES})
    batch = [P.ExperienceTuple(i, P.pack_solution(z["snaps"][i]), int(z["actions"][i]), 0.0)
             for i in range(B)]

    def worker(comm):
        part = P.partition_rows(n, 1)[0]
        adam = P.AdamState.create(params, lr=1e-5)
        state = P.tuples_to_graphs(batch, dataset, part, dtype=dtype)
        targets = P.batch_targets(batch, dataset, params, comm, part, 0.9).astype(dtype)
        losses, g0 = [], None
        for it in range(tau):
            loss, grads = P.loss_and_gradients(state, z["actions"], targets, params, comm)
            g0 = g0 or grads
            P.adam_step(params, grads, adam)
            losses.append(loss)
        return targets, losses, g0, adam
    targets, losses, g0, adam = P.run_workers(1, worker)[0]
    # targets come from the bit-exact forward: identical
    assert np.array_equal(targets, z["targets"])
    assert scale_error(losses, z["losses"]).max() < tol
    for k in P.PARAM_NAMES:
        assert scale_error(g0[k], z[f"g0_{k}"]).max() < tol, k
        assert scale_error(getattr(params, k), z[f"p1_{k}"]).max() < tol, k


def test_cfg2_device_tau_loop_matches_reference():
    """BASELINE configs[1] through train_step's device-resident tau loop
    (policy.train_iterations): per-iteration losses and the post-Adam
    parameters and moments after tau = 4 match the reference's at 1e-4."""
    from paper_2105_08764_b200.policy import train_iterations
    path = GOLD / "train_cfg2_ba10k_b32_k64_l5.npz"
    if not path.exists():
        pytest.skip("golden fixture not generated")
    z = np.load(path)
    n, m, B, K, L, tau = (int(z[k]) for k in ("n", "m", "B", "K", "L", "tau"))
    dataset = [P.generate_ba(n, m, 100 + i) for i in range(B)]
    params = P.PolicyParams(num_layers=L, **{k: z[f"p0_{k}"].copy() for k in P.PARAM_NAMES})
    batch = [P.ExperienceTuple(i, P.pack_solution(z["snaps"][i]), int(z["actions"][i]), 0.0)
             for i in range(B)]

    def worker(comm):
        part = P.partition_rows(n, 1)[0]
        adam = P.AdamState.create(params, lr=1e-5)
        state = P.tuples_to_graphs(batch, dataset, part)
        targets = P.batch_targets(batch, dataset, params, comm, part, 0.9).astype(np.float32)
        losses = train_iterations(state, z["actions"], targets, params, adam, tau, comm)
        return targets, losses, adam
    targets, losses, adam = P.run_workers(1, worker)[0]
    assert np.array_equal(targets, z["targets"])
    assert scale_error(losses, z["losses"]).max() < 1e-4
    for k in P.PARAM_NAMES:
        assert scale_error(getattr(params, k), z[f"p1_{k}"]).max() < 1e-4, k
        assert scale_error(adam.m[k], z[f"m_{k}"]).max() < 1e-4, k
        assert scale_error(adam.v[k], z[f"v_{k}"]).max() < 1e-4, k


@pytest.mark.parametrize("dtype,tol", [(np.float32, 1e-4), (np.float64, 1e-9)])
@pytest.mark.parametrize("K,L,B", [(8, 2, 3), (32, 3, 2), (64, 5, 4)])
def test_loss_and_gradients_vs_port(dtype, tol, K, L, B):
    rng = np.random.default_rng(K * 10 + L)
    n = 400
    graphs = [P.generate_ba(n, 3, 50 + i) for i in range(B)]
    sols = (rng.random((B, n)) < 0.15).astype(np.uint8)
    params = P.PolicyParams.initialize(K, L, seed=K, dtype=dtype, orientation="symmetric")
    ps = port.ResidualState([g.edge_array for g in graphs], n, solutions=sols, dtype=dtype)
    actions = np.array([int(np.flatnonzero(ps.cand[b])[rng.integers(
        np.count_nonzero(ps.cand[b]))]) for b in range(B)])
    targets = rng.normal(size=B).astype(dtype)

    def worker(comm):
        st = P.PartitionedState(graphs, P.partition_rows(n, 1)[0], solutions=sols, dtype=dtype)
        return P.loss_and_gradients(st, actions, targets, params, comm)
    loss, grads = P.run_workers(1, worker)[0]
    loss_o, grads_o = port.loss_and_grads(ps, actions, targets, params.as_dict(), L)
    assert abs(loss - loss_o) <= tol * max(1.0, abs(loss_o))
    for k in P.PARAM_NAMES:
        assert scale_error(grads[k], grads_o[k]).max() < tol, k


def test_adam_bitwise_vs_port():
    params = P.PolicyParams.initialize(16, 2, seed=3)
    rng = np.random.default_rng(1)
    theta = {k: v.copy() for k, v in params.as_dict().items()}
    m = {k: np.zeros_like(v) for k, v in theta.items()}
    v = {k: np.zeros_like(x) for k, x in theta.items()}
    adam = P.AdamState.create(params, lr=1e-3)
    step = 0

    def run(grads):
        return P.run_workers(1, lambda comm: P.adam_step(params, grads, adam))[0]
    for it in range(3):
        grads = {k: (rng.normal(size=x.shape) * 10.0 ** rng.integers(-3, 8)).astype(np.float32)
                 for k, x in theta.items()}
        run(grads)
        step = port.adam(theta, grads, m, v, step, 1e-3)
    for k in P.PARAM_NAMES:
        assert np.array_equal(getattr(params, k), theta[k]), k
        assert np.array_equal(adam.m[k], m[k]) and np.array_equal(adam.v[k], v[k])


def test_loss_and_gradients_with_hub_rows_vs_port():
    base = P.generate_ba(6000, 4, 5)
    extra = np.stack([np.full(5000, 7), np.arange(1000, 6000)], axis=1)
    g = P.Graph(6000, np.concatenate([base.edge_array, extra]))
    rng = np.random.default_rng(3)
    B, n = 2, 6000
    sols = (rng.random((B, n)) < 0.05).astype(np.uint8)
    sols[:, 7] = 0
    params = P.PolicyParams.initialize(64, 4, seed=5, orientation="symmetric")
    ps = port.ResidualState([g.edge_array] * B, n, solutions=sols)
    actions = np.array([7, int(np.flatnonzero(ps.cand[1])[3])])
    targets = rng.normal(size=B).astype(np.float32)

    def worker(comm):
        st = P.PartitionedState([g] * B, P.partition_rows(n, 1)[0], solutions=sols)
        assert st.n_hub >= 1
        return P.loss_and_gradients(st, actions, targets, params, comm)
    loss, grads = P.run_workers(1, worker)[0]
    loss_o, grads_o = port.loss_and_grads(ps, actions, targets, params.as_dict(), 4)
    assert abs(loss - loss_o) <= 1e-4 * max(1.0, abs(loss_o))
    for k in P.PARAM_NAMES:
        assert scale_error(grads[k], grads_o[k]).max() < 1e-4, k


def test_ffma_backward_path_vs_port():
    """The FFMA layer-backward kernel (S2V_BWD_TC=0; the default K = 64 path
    is the tcgen05 split-TF32 kernel): same K=64 parity cases, run in a child
    process because the path is chosen once per process."""
    import os
    import subprocess
    import sys
    here = Path(__file__).resolve().parent
    env = dict(os.environ, S2V_BWD_TC="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        str(here / "test_gpu_train.py"), "-k",
                        "(vs_port and 64) or hub or ba1000", "-m", "gpu"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_device_tau_loop_equals_host_loop():
    """train_step's device-resident tau loop (policy.train_iterations) gives
    the parameters, moments, step count and losses of the host-driven
    loss_and_gradients + adam_step loop, bit for bit."""
    from paper_2105_08764_b200.policy import train_iterations
    gs = [P.generate_ba(3000, 4, 40 + i) for i in range(4)]
    rng = np.random.default_rng(3)
    sol = (rng.random((4, 3000)) < 0.1).astype(np.uint8)
    targets = rng.normal(size=4).astype(np.float32)

    def run(device_loop):
        def worker(comm):
            part = P.partition_rows(3000, 1)[0]
            st = P.PartitionedState(gs, part, solutions=sol)
            acts = np.array([int(np.flatnonzero(st.cand[b])[7]) for b in range(4)])
            params = P.PolicyParams.initialize(64, 5, seed=2)
            adam = P.AdamState.create(params, lr=1e-3)
            if device_loop:
                losses = train_iterations(st, acts, targets, params, adam, 3, comm)
            else:
                losses = []
                for _ in range(3):
                    loss, grads = P.loss_and_gradients(st, acts, targets, params, comm)
                    P.adam_step(params, grads, adam)
                    losses.append(loss)
            return losses, params.as_dict(), adam.m, adam.v, adam.step
        return P.run_workers(1, worker)[0]

    got, want = run(True), run(False)
    assert got[0] == want[0] and got[4] == want[4] == 3
    for a, b in zip(got[1:4], want[1:4]):
        for name in P.PARAM_NAMES:
            assert np.array_equal(a[name], b[name]), name


def test_device_tau_loop_rejects_non_finite():
    """A target that overflows the gradients: the step is rejected (params,
    moments and step count untouched) with adam_step's ValueError."""
    from paper_2105_08764_b200.policy import train_iterations
    g = P.generate_ba(2000, 4, 5)

    def worker(comm):
        part = P.partition_rows(2000, 1)[0]
        st = P.PartitionedState([g], part)
        params = P.PolicyParams.initialize(64, 5, seed=0)
        before = {k: v.copy() for k, v in params.as_dict().items()}
        adam = P.AdamState.create(params, lr=1e-3)
        act = np.array([int(np.flatnonzero(st.cand[0])[0])])
        try:
            train_iterations(st, act, np.array([3e38], np.float32), params, adam, 2, comm)
        except ValueError as e:
            msg = str(e)
        else:
            msg = ""
        same = all(np.array_equal(before[k], v) for k, v in params.as_dict().items())
        return msg, same, adam.step
    msg, same, step = P.run_workers(1, worker)[0]
    assert "non-finite gradient" in msg and same and step == 0


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("B,n,K", [(1, 5, 8), (2, 1003, 64), (3, 4099, 16), (2, 70001, 64),
                                   (1, 2049, 2)])
def test_theta2_einsum_order_bitwise(dtype, B, n, K):
    """s2v_theta2_einsum reproduces np.einsum("bkv,bv->k") (policy.py:305-306)
    bit for bit on terms with heavy cancellation, tails included: with
    deg = 1 the einsum's products are the terms themselves."""
    import torch
    from paper_2105_08764_b200 import _lib
    from paper_2105_08764_b200.device import stream_ptr
    rng = np.random.default_rng(B * n + K)
    X = (rng.normal(size=(B, K, n)) * np.exp(rng.normal(size=(B, K, n)) * 4)).astype(dtype)
    want = np.einsum("bkv,bv->k", X, np.ones((B, n), dtype))
    G = 32 // np.dtype(dtype).itemsize
    ng = (K + G - 1) // G
    lay = np.zeros((B, ng * G, n), dtype)
    lay[:, :K] = X
    lay = np.ascontiguousarray(lay.reshape(B, ng, G, n).transpose(0, 1, 3, 2))
    g = P.Graph(n, [(i, i + 1) for i in range(n - 1)])

    def worker(comm):
        st = P.PartitionedState([g] * B, P.partition_rows(n, 1)[0], dtype=dtype)
        lib = _lib.load()
        dt = _lib.S2V_F32 if dtype == np.float32 else _lib.S2V_F64
        assert lib.s2v_theta2_terms_bytes(dt, st.shard_ref(), K) == lay.nbytes
        t2c = torch.from_numpy(lay.ravel()).to(st.device)
        tot = torch.empty(B * K, dtype=t2c.dtype, device=st.device)
        out = torch.empty(K, dtype=torch.float64, device=st.device)
        _lib.call("s2v_theta2_einsum", dt, st.shard_ref(), K, t2c.data_ptr(), tot.data_ptr(),
                  out.data_ptr(), stream_ptr())
        return out.cpu().numpy()
    got = P.run_workers(1, worker)[0]
    assert np.array_equal(got.astype(dtype), want)
