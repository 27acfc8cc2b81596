"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle on the same seeded inputs.

Bars: bit-exact for init, broadcast, the fused average +
update (K6) and integer/index work; max-norm relative error per tensor within
1e-5 (the fp32 tier: MTX_FP32 SIMT and MTX_3XTF32 tensor cores) for gradients,
losses, velocities and weight changes, every step checked from the GPU's own state.
"""
from __future__ import annotations

import numpy as np
import pytest

import mtx_synth as S
import oracle
from tests._parity import step_errors
from tests._util import GRAD_TOL, TOL, digest_np, maxrel, per_tensor_maxrel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1704_04560_b200 as P  # noqa: E402  (loads libmtx.so; raises if missing)
from paper_1704_04560_b200 import mtx  # noqa: E402

PRECISIONS = [P.MTX_FP32] + ([P.MTX_3XTF32, P.MTX_3XF16] if "tcgen05" in mtx.mtx_build_info() else [])


def small_cfg(name, **kw):
    c = dict(S.CONFIGS[name])
    c.update(kw)
    return c


def make(cfg, precision=P.MTX_FP32, **kw):
    r = P.Replica(cfg, precision=precision, **kw)
    return r


# ----------------------------------------------------------------------------- K6 bit-exact
@pytest.mark.parametrize("n", [1024, 1 << 20, (1 << 20) + 3, 61_100_840 // 8 + 1])
@pytest.mark.parametrize("mu", [0.9, 0.0])
def test_fused_avg_update_bit_exact(n, mu):
    r = make(small_cfg("cfg1", B=4, P=1))
    try:
        G = S.cfg5_grad_random(1, 0, n)
        w = S.cfg5_params(1, n)
        v = S.cfg5_velocity(1, n)
        dev = lambda a: torch.from_numpy(a.copy()).cuda()
        Gd, wd, vd = dev(G), dev(w), dev(v)
        torch.cuda.synchronize()
        mtx.mtx_allreduce_avg(r.ctx, Gd.data_ptr(), wd.data_ptr(), vd.data_ptr() if mu else None, n, 0.01, mu, 1,
                              r.s)
        r.sync()
        wo, vo = w.copy(), v.copy() if mu else np.zeros(n, np.float32)
        oracle.avg_update(G, wo, vo, 1, 0.01, mu)
        assert np.array_equal(wd.cpu().numpy().view(np.uint32), wo.view(np.uint32))
        if mu:
            assert np.array_equal(vd.cpu().numpy().view(np.uint32), vo.view(np.uint32))
    finally:
        r.close()


def test_sync_update_single_rank_bit_exact():
    """mtx_sync_update at P = 1: G = the injected gradient; w, v bit-exact with the oracle's fp32 update."""
    cfg = small_cfg("cfg2")
    net = oracle.Net.from_cfg(cfg)
    n = oracle.param_count(net)
    rng = np.random.default_rng(9)
    g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    w0 = oracle.init_params(net, 42)
    v0 = (rng.standard_normal(n) * 1e-3).astype(np.float32)
    r = make(cfg, bucket_bytes=256 << 10)
    try:
        r.bcast()
        r.set(P.MTX_BUF_PARAMS, w0)
        r.set(P.MTX_BUF_VELOCITY, v0)
        r.set(P.MTX_BUF_GRADS, g)
        mtx.mtx_sync_update(r.ctx, r.s)
        wo, vo = w0.copy(), v0.copy()
        oracle.avg_update(g, wo, vo, 1, cfg["lr"], cfg["mu"])
        assert np.array_equal(r.get(P.MTX_BUF_GRADS).view(np.uint32), g.view(np.uint32))
        assert np.array_equal(r.get(P.MTX_BUF_PARAMS).view(np.uint32), wo.view(np.uint32))
        assert np.array_equal(r.get(P.MTX_BUF_VELOCITY).view(np.uint32), vo.view(np.uint32))
    finally:
        r.close()


def test_fused_update_flags_non_finite():
    r = make(small_cfg("cfg1", B=4, P=1))
    try:
        g = torch.zeros(1024, device="cuda")
        g[17] = float("nan")
        w = torch.zeros(1024, device="cuda")
        v = torch.zeros(1024, device="cuda")
        mtx.mtx_allreduce_avg(r.ctx, g.data_ptr(), w.data_ptr(), v.data_ptr(), 1024, 0.1, 0.9, 1, r.s)
        with pytest.raises(P.MtxError) as e:
            r.get()
        assert e.value.status == 6  # MTX_ERR_NUMERIC
    finally:
        r.close()


# ----------------------------------------------------------------------------- init + broadcast
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg4"])
def test_init_bit_exact(name):
    cfg = small_cfg(name, B=8)
    r = make(cfg, init_seed=42)
    try:
        want = oracle.init_params(oracle.Net.from_cfg(cfg), 42)
        got = r.get()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
        # single rank: broadcast keeps the bits and zeroes the velocity
        r.bcast()
        assert np.array_equal(r.get().view(np.uint32), want.view(np.uint32))
        assert not r.get(P.MTX_BUF_VELOCITY).any()
        assert r.digest() == digest_np(r.get(), r.get(P.MTX_BUF_VELOCITY))
    finally:
        r.close()


# ----------------------------------------------------------------------------- one-step and trajectory parity
def _gpu_run(cfg, X, y, steps, precision, start=None, start_step=0, **kw):
    """GPU steps through the C-ABI; per step (loss, G, w after, v after)."""
    r = make(cfg, precision=precision, **kw)
    try:
        r.bcast()
        if start is not None:
            r.set(P.MTX_BUF_PARAMS, start)
        r.shard(X, y)
        r.step_idx = start_step
        out = []
        for _ in range(steps):
            loss = r.step(want_loss=True)
            out.append((loss, r.get(P.MTX_BUF_GRADS), r.get(P.MTX_BUF_PARAMS), r.get(P.MTX_BUF_VELOCITY)))
        return out
    finally:
        r.close()


def _check_step(cfg, X, y, precision, step, start, **kw):
    """One step from identical params: G, loss, velocity and weight change vs the oracle (P = 1)."""
    net = oracle.Net.from_cfg(cfg)
    rec, = _gpu_run(cfg, X, y, 1, precision, start=start, start_step=step, **kw)
    e = step_errors(net, cfg, X, y, step, start, np.zeros_like(start), rec)
    assert max(e.values()) <= GRAD_TOL[precision], e


@pytest.mark.parametrize("precision", PRECISIONS)
def test_cfg1_one_step(precision):
    cfg = small_cfg("cfg1", B=64)
    X, y = S.mnist_like(1, 1000)
    start = oracle.init_params(oracle.Net.from_cfg(cfg), 42)
    _check_step(cfg, X, y, precision, 0, start)
    _check_step(cfg, X, y, precision, 15, start)  # window wraps around n = 1000


def _check_trajectory(cfg, X, y, steps, precision, **kw):
    """Every step of a GPU trajectory within the fp32 tier of the oracle step from the GPU's own state,
    and the whole trajectory (losses, final weights) within it of the oracle's own trajectory."""
    net = oracle.Net.from_cfg(cfg)
    recs, w_ref, _ = oracle.train(net, X, y, cfg["B"], 1, steps, cfg["lr"], cfg["mu"], 42)
    gpu = _gpu_run(cfg, X, y, steps, precision, **kw)
    w0 = oracle.init_params(net, 42)
    v0 = np.zeros_like(w0)
    tol = TOL[precision]
    for t, (rec, g) in enumerate(zip(recs, gpu)):
        e = step_errors(net, cfg, X, y, t, w0, v0, g)
        assert max(e.values()) <= GRAD_TOL[precision], (t, e)
        assert abs(g[0] - rec.loss) <= tol * abs(rec.loss), t
        w0, v0 = g[2], g[3]
    assert maxrel(gpu[-1][2], w_ref) <= tol


@pytest.mark.parametrize("precision", PRECISIONS)
def test_cfg1_trajectory_five_steps(precision):
    """configs[0]: MLP 784-128-10, B=64, 5 SGD steps (run at P=1 on one GPU)."""
    _check_trajectory(small_cfg("cfg1", B=64), *S.mnist_like(1, 1000), 5, precision)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_cfg2_one_step_and_wrap(precision):
    """configs[1] model (784-512-512-10, B=512, momentum) at full batch; step 117 wraps n=60000."""
    cfg = small_cfg("cfg2")
    X, y = S.mnist_like(1, 60000)
    start = oracle.init_params(oracle.Net.from_cfg(cfg), 42)
    _check_step(cfg, X, y, precision, 0, start)
    _check_step(cfg, X, y, precision, 117, start)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_cfg2_small_buckets_two_steps(precision):
    """Per-layer buckets: each bucket's update must not race the dgrad that still reads W_l."""
    _check_trajectory(small_cfg("cfg2"), *S.mnist_like(1, 4096), 2, precision, bucket_bytes=64 << 10)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_cfg4_shape_one_step(precision):
    """configs[3] model 28-1024x4-2 (K = 28 ragged, N = 2 head) at a batch the oracle finishes in seconds."""
    cfg = small_cfg("cfg4", B=96, n=5000)
    X, y = S.higgs_like(1, 5000)
    start = oracle.init_params(oracle.Net.from_cfg(cfg), 42)
    _check_step(cfg, X, y, precision, 3, start)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_ragged_mlp_one_step(precision):
    """Odd widths and batch: every tile edge ragged."""
    cfg = dict(kind="mlp", dims=[37, 71, 130, 3], data="mnist", n=500, B=75, lr=0.05, mu=0.9)
    rng = np.random.default_rng(0)
    X = rng.standard_normal((500, 37)).astype(np.float32)
    y = rng.integers(0, 3, 500).astype(np.int32)
    start = oracle.init_params(oracle.Net.from_cfg(cfg), 42)
    _check_step(cfg, X, y, precision, 4, start)


@pytest.mark.parametrize("precision", PRECISIONS)
@pytest.mark.parametrize("dims,B", [([20, 72, 96, 3], 75), ([28, 200, 136, 2], 300)])
def test_short_input_mlp_ragged(precision, dims, B):
    """A <= 64-feature input layer feeding tensor-core GEMMs (3xF16: the CUDA-core fwd_smallk forward with planes and
    ReLU bits) with ragged rows and a ragged last column block, and the lean hidden tensors after it."""
    cfg = dict(kind="mlp", dims=dims, data="higgs", n=B + 200, B=B, lr=0.05, mu=0.9)
    rng = np.random.default_rng(sum(dims) + B)
    X = rng.standard_normal((B + 200, dims[0])).astype(np.float32)
    y = rng.integers(0, dims[-1], B + 200).astype(np.int32)
    start = oracle.init_params(oracle.Net.from_cfg(cfg), 42)
    _check_step(cfg, X, y, precision, 3, start)


@pytest.mark.parametrize("precision", PRECISIONS[1:] or PRECISIONS)
@pytest.mark.parametrize("C,d,B", [(10, 71, 75), (2, 71, 75), (10, 64, 2100), (2, 33, 2100), (1, 40, 75),
                                   (5, 130, 75), (16, 129, 75)])
def test_head_class_counts(C, d, B, precision):
    """The fused head's instances: exact C = 2 / 10 (HIGGS, MNIST/CIFAR), generic C <= 4 / <= 16,
    vector and scalar (d % 4 != 0) row loads, and the > 2048-row launch shape; B is ragged."""
    cfg = dict(kind="mlp", dims=[24, d, C], data="mnist", n=B + 50, B=B, lr=0.05, mu=0.9)
    rng = np.random.default_rng(C * 1000 + d)
    X = rng.standard_normal((B + 50, 24)).astype(np.float32)
    y = rng.integers(0, C, B + 50).astype(np.int32)
    start = oracle.init_params(oracle.Net.from_cfg(cfg), 42)
    _check_step(cfg, X, y, precision, 1, start)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_cnn_lenet_one_step(precision):
    """configs[2] model (LeNet on CIFAR-shaped NHWC 32x32x3) at a batch the oracle finishes in seconds;
    step 3 wraps the window (n = 200, B = 64)."""
    cfg = small_cfg("cfg3", B=64, n=200)
    X, y = S.cifar_like(1, 200)
    start = oracle.init_params(oracle.Net.from_cfg(cfg), 42)
    _check_step(cfg, X, y, precision, 0, start)
    _check_step(cfg, X, y, precision, 3, start)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_cnn_mini_one_step(precision):
    """Odd geometry: two conv stages (3x3 then 2x2, odd spatial sizes so pooling drops edges)."""
    cfg = dict(kind="cnn", in_hwc=(13, 13, 2), conv=[(3, 5), (2, 7)], fc=[9, 4], data="cifar", n=100, B=30,
               lr=0.05, mu=0.9)
    rng = np.random.default_rng(5)
    X = rng.standard_normal((100, 13, 13, 2)).astype(np.float32)
    y = rng.integers(0, 4, 100).astype(np.int32)
    start = oracle.init_params(oracle.Net.from_cfg(cfg), 42)
    _check_step(cfg, X, y, precision, 1, start)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_full_size_cfg4_replicated_rows(precision):
    """Full cfg4 launch configuration (B = 8192) on a dataset of 128 copies of 64 rows: the
    mean gradient over 8192 rows equals the oracle's over the 64 distinct rows."""
    cfg = small_cfg("cfg4")
    X64, y64 = S.higgs_like(1, 64)
    X = np.tile(X64, (128, 1))
    y = np.tile(y64, 128)
    net = oracle.Net.from_cfg(cfg)
    start = oracle.init_params(net, 42)
    (loss, G, w1, _), = _gpu_run(cfg, X, y, 1, precision, start=start)
    g_ref, lsum = oracle.local_grad(net, start.astype(np.float64), X64, y64, 64, 0, 0, 1)
    assert max(per_tensor_maxrel(G, g_ref, oracle.tensor_table(net))) <= 1e-5
    assert abs(loss - lsum / 64) <= 1e-5 * abs(lsum / 64)


@pytest.mark.parametrize("precision", PRECISIONS)
def test_full_size_cfg3_replicated_rows(precision):
    """Full cfg3 launch configuration (LeNet, B = 1024, the conv kernels' bench grid) on a dataset of
    64 copies of 16 CIFAR-shaped images: the mean gradient over 1024 rows equals the oracle's over the
    16 distinct images, and one momentum step lands on the oracle's weights."""
    cfg = small_cfg("cfg3", n=1024)
    X16, y16 = S.cifar_like(1, 16)
    X = np.tile(X16, (64, 1, 1, 1))
    y = np.tile(y16, 64)
    net = oracle.Net.from_cfg(cfg)
    start = oracle.init_params(net, 42)
    (loss, G, w1, _), = _gpu_run(cfg, X, y, 1, precision, start=start)
    g_ref, lsum = oracle.local_grad(net, start.astype(np.float64), X16, y16, 16, 0, 0, 1)
    tab = oracle.tensor_table(net)
    assert max(per_tensor_maxrel(G, g_ref, tab)) <= 1e-5
    assert abs(loss - lsum / 16) <= 1e-5 * abs(lsum / 16)
    w_ref = start.astype(np.float64).copy()
    oracle.avg_update(g_ref, w_ref, np.zeros_like(w_ref), 1, cfg["lr"], cfg["mu"])
    assert max(per_tensor_maxrel(w1, w_ref, tab)) <= 1e-5


# ----------------------------------------------------------------------------- host-input path, state machine
def test_host_staged_step_matches_resident():
    cfg = small_cfg("cfg2")
    X, y = S.mnist_like(1, 4096)
    r1, r2 = make(cfg), make(cfg)
    try:
        for r in (r1, r2):
            r.bcast()
        r1.shard(X, y)
        for t in range(3):
            l1 = r1.step(want_loss=True)
            (b0, b1), (n0, n1) = mtx.mtx_batch_slice(4096, 512, t, 0, 1)
            idx = np.r_[b0:b0 + n0, b1:b1 + n1]
            Xr = np.ascontiguousarray(X[idx])
            yr = np.ascontiguousarray(y[idx])
            l2 = r2.step_host(Xr, yr)
            assert l1 == l2
        assert np.array_equal(r1.get().view(np.uint32), r2.get().view(np.uint32))
    finally:
        r1.close()
        r2.close()


@pytest.mark.parametrize("precision", PRECISIONS)
def test_pipelined_host_steps_match_synchronous(precision):
    """mtx_train_step_host_async (double-buffered landing, copy of step t+1 overlapping step t) gives the
    bit-identical trajectory of mtx_train_step_host on the same rows, and mtx_sync reports its last loss."""
    import torch
    cfg = small_cfg("cfg2")
    X, y = S.mnist_like(1, 4096)
    r1, r2 = make(cfg, precision=precision), make(cfg, precision=precision)
    try:
        for r in (r1, r2):
            r.bcast()
        rows = []
        for t in range(5):
            (b0, b1), (n0, n1) = mtx.mtx_batch_slice(4096, 512, t, 0, 1)
            idx = np.r_[b0:b0 + n0, b1:b1 + n1]
            rows.append((torch.from_numpy(np.ascontiguousarray(X[idx])).pin_memory(),
                         torch.from_numpy(np.ascontiguousarray(y[idx])).pin_memory()))
        losses = [r1.step_host(Xr.numpy(), yr.numpy()) for Xr, yr in rows]
        for Xr, yr in rows:
            r2.step_host_async(Xr.numpy(), yr.numpy())
        last = r2.sync_host()
        assert last == losses[-1]
        assert np.array_equal(r1.get().view(np.uint32), r2.get().view(np.uint32))
    finally:
        r1.close()
        r2.close()


def test_state_machine_and_errors():
    cfg = small_cfg("cfg1", B=64)
    r = make(cfg)
    try:
        with pytest.raises(P.MtxError) as e:
            r.step()
        assert e.value.status == 2  # MTX_ERR_STATE: no broadcast / dataset yet
        r.bcast()
        with pytest.raises(P.MtxError) as e:
            mtx.mtx_shard_data(r.ctx, 1, 1, 1000, 783, 0, r.ws.data_ptr(), 10, r.s)
        assert e.value.status == 3  # MTX_ERR_SHAPE
        X, y = S.mnist_like(1, 32)
        with pytest.raises(P.MtxError) as e:
            r.shard(X, y)  # B = 64 > n = 32
        assert e.value.status == 1
    finally:
        r.close()
    with pytest.raises(P.MtxError) as e:
        P.Replica(small_cfg("cfg1", B=63), world=2, rank=0, uid=bytes(128))  # B mod P != 0
    assert e.value.status == 1


def test_nan_params_raise_numeric():
    cfg = small_cfg("cfg1", B=64)
    X, y = S.mnist_like(1, 1000)
    r = make(cfg)
    try:
        r.bcast()
        w = r.get()
        w[-1] = np.nan  # b_L: every logit row turns NaN (a NaN behind a ReLU would be clipped by max(z, 0))
        r.set(P.MTX_BUF_PARAMS, w)
        r.shard(X, y)
        with pytest.raises(P.MtxError) as e:
            r.step(want_loss=True)
        assert e.value.status == 6
    finally:
        r.close()


def test_graph_launch_count_and_determinism():
    cfg = small_cfg("cfg2")
    X, y = S.mnist_like(1, 8192)
    outs = []
    for _ in range(2):
        r = make(cfg)
        try:
            r.bcast()
            r.shard(X, y)
            for _ in range(4):
                r.step()
            outs.append((r.get().tobytes(), r.digest()))
            assert mtx.mtx_launches_per_step(r.ctx) > 0
        finally:
            r.close()
    assert outs[0] == outs[1]  # run-to-run bitwise determinism (no float atomics)
