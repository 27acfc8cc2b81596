"""Pins for the CPU oracle (``-m "not gpu"``): each test checks the oracle against
something other than itself -- published test vectors, worked values from
SPEC.md, exact rational arithmetic, finite differences, an independent library
(torch CPU autograd in float64), invariants of the method (P-rank = sequential,
bit-identical replicas) and brute-force sweeps.  DESIGN.md §"Oracle pins" maps
each oracle function to the tests here.
"""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np
import pytest

import mtx_synth as S
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------- O1 generator
def test_splitmix64_known_answer_vector():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "splitmix64_kat.txt")) if l.strip() and l[0] != "#"]
    assert len(rows) == 4
    for seed, k, hexval in rows:
        want = int(hexval, 16)
        assert oracle.splitmix64(int(seed), int(k)) == want
        assert int(S.splitmix64(int(seed), np.array([int(k)]))[0]) == want


def test_synth_shapes_and_statistics():
    X, y = S.mnist_like(1, 2000)
    assert X.shape == (2000, 784) and X.dtype == np.float32 and y.dtype == np.int32
    assert X.min() >= 0 and X.max() <= 1 and set(np.unique(y)) == set(range(10))
    nz = (X > 0).mean()
    assert 0.15 < nz < 0.25  # ~19% strokes, like MNIST
    Xc, yc = S.cifar_like(1, 300)
    assert Xc.shape == (300, 32, 32, 3) and 0.3 < Xc.mean() < 0.7
    Xh, yh = S.higgs_like(1, 20000)
    assert Xh.shape == (20000, 28) and abs(yh.mean() - 0.53) < 0.02
    assert 1.0 < Xh[yh == 0].std() < 1.3
    # determinism: same seed, same bytes; different seed, different bytes
    assert S.mnist_like(1, 50)[0].tobytes() == S.mnist_like(1, 50)[0].tobytes()
    assert S.mnist_like(2, 50)[0].tobytes() != S.mnist_like(1, 50)[0].tobytes()


def test_cfg5_dyadic_values_are_exactly_summable():
    g = np.stack([S.cfg5_grad_dyadic(1, r, 4096) for r in range(8)]).astype(np.float64)
    ints = g * 2 ** 8
    assert np.all(ints == np.round(ints)) and np.abs(ints).max() <= 2 ** 20
    # any summation order of 8 such values is exact in fp32 (|sum| < 2^24 units of 2^-8)
    f = np.stack([S.cfg5_grad_dyadic(1, r, 4096) for r in range(8)])
    assert np.array_equal(oracle.fold(f).astype(np.float64), ints.sum(0) / 2 ** 8)
    assert np.array_equal(oracle.fold(f[::-1].copy()), oracle.fold(f))


# ----------------------------------------------------------------------------- O2 init
def test_init_glorot_statistics_and_determinism():
    net = oracle.Net("mlp", [784, 512, 512, 10])
    w = oracle.init_params(net, 42)
    assert w.dtype == np.float32
    for t, (off, size) in enumerate(oracle.tensor_table(net)):
        x = w[off:off + size].astype(np.float64)
        if t % 2 == 1:  # biases are zero
            assert np.all(x == 0)
            continue
        fi, fo = net.dims[t // 2], net.dims[t // 2 + 1]
        # Glorot & Bengio (2010): Var(w) = 2 / (fan_in + fan_out), uniform on a symmetric range
        var_want = 2.0 / (fi + fo)
        assert abs(x.var() / var_want - 1) < 0.03, (t, x.var(), var_want)
        assert abs(x.mean()) < 4 * math.sqrt(var_want / size)
        assert abs(x.max() + x.min()) < 0.01 * x.max()  # symmetric support
    assert oracle.init_params(net, 42).tobytes() == w.tobytes()
    assert oracle.init_params(net, 43).tobytes() != w.tobytes()


def test_init_conv_fans():
    net = oracle.Net("cnn", [], (32, 32, 3), [(5, 6), (5, 16)], [120, 84, 10])
    w = oracle.init_params(net, 7)
    off, size = oracle.tensor_table(net)[0]  # conv1 W [5][5][3][6]: fan_in 75, fan_out 150
    x = w[off:off + size].astype(np.float64)
    assert abs(x.var() / (2.0 / (75 + 150)) - 1) < 0.15


def test_lenet_parameter_count():
    # 5*5*3*6+6, 5*5*6*16+16, 400*120+120, 120*84+84, 84*10+10
    net = oracle.Net("cnn", [], (32, 32, 3), [(5, 6), (5, 16)], [120, 84, 10])
    assert [s for _, s in oracle.tensor_table(net)] == [450, 6, 2400, 16, 48000, 120, 10080, 84, 840, 10]
    assert oracle.param_count(net) == 62006
    assert oracle.param_count(oracle.Net("mlp", [28, 1024, 1024, 1024, 1024, 2])) == 3180546
    assert oracle.param_count(oracle.Net("mlp", [784, 512, 512, 10])) == 669706


# ----------------------------------------------------------------------------- O4 shard
def test_batch_slice_worked_values():
    # n=100, B=8, step 0, p=4 -> 2,2,2,2 covering 0..7
    ids = []
    for r in range(4):
        (b0, b1), (l0, l1) = oracle.batch_slice(100, 8, 0, r, 4)
        assert l0 + l1 == 2
        ids += list(range(b0, b0 + l0)) + list(range(b1, b1 + l1))
    assert ids == list(range(8))
    # step 13: window starts at 104 mod 100 = 4
    (b0, _), _ = oracle.batch_slice(100, 8, 13, 0, 4)
    assert b0 == 4
    # A1: B mod P != 0 is rejected (SPEC's B=5, p=4 case is out of scope for this build)
    with pytest.raises(ValueError):
        oracle.batch_slice(100, 5, 0, 0, 4)


def test_batch_slice_exhaustive_partition():
    for n in (1, 2, 3, 7, 10, 64, 100):
        for P in (1, 2, 3, 4, 8, 16):
            for b in (1, 2, 3, 5):
                B = b * P
                if B > n:  # a window larger than the dataset is rejected
                    with pytest.raises(ValueError):
                        oracle.batch_slice(n, B, 0, 0, P)
                    continue
                for step in (0, 1, 5, 13, 117):
                    window = [(step * B + k) % n for k in range(B)]
                    got = []
                    for r in range(P):
                        (b0, b1), (l0, l1) = oracle.batch_slice(n, B, step, r, P)
                        piece = list(range(b0, b0 + l0)) + list(range(b1, b1 + l1))
                        assert len(piece) == b and all(0 <= i < n for i in piece)
                        got += piece
                    assert got == window, (n, P, B, step)


# ----------------------------------------------------------------------------- O5-O7 math
def test_relu_affine_worked_value():
    net = oracle.Net("mlp", [2, 2, 2])
    p = np.zeros(oracle.param_count(net))
    p[0:4] = [1, 0, 0, 1]  # W_1 = I, b_1 = 0
    a1 = oracle.mlp_activations(net, p, np.array([[1, -2]], np.float32), np.array([0], np.int32), 1)
    assert a1.tolist() == [[1.0, 0.0]]


def test_softmax_xent_worked_values():
    net = oracle.Net("mlp", [3, 2])  # one layer: logits = x W + b
    p = np.zeros(oracle.param_count(net))
    X = np.array([[0.5, -1.0, 2.0]], np.float32)
    g, loss = oracle.batch_grad(net, p, X, np.array([0], np.int32))
    assert abs(loss - math.log(2)) < 1e-15
    db = g[6:8]
    assert db.tolist() == [-0.5, 0.5]
    dW = g[:6].reshape(3, 2)
    assert np.array_equal(dW, X.T.astype(np.float64) @ np.array([[-0.5, 0.5]]))


def _fd_check(net, X, y, rng, n_coords=None):
    N = oracle.param_count(net)
    p = rng.standard_normal(N) * 0.5
    g, _ = oracle.batch_grad(net, p, X, y)
    b = X.shape[0]
    h = 1e-6
    coords = range(N) if n_coords is None else rng.choice(N, n_coords, replace=False)
    worst = 0.0
    for e in coords:
        pp, pm = p.copy(), p.copy()
        pp[e] += h
        pm[e] -= h
        lp = oracle.batch_grad(net, pp, X, y, want_grad=False)[1] / b
        lm = oracle.batch_grad(net, pm, X, y, want_grad=False)[1] / b
        fd = (lp - lm) / (2 * h)
        err = abs(fd - g[e]) / max(abs(fd), abs(g[e]), 1e-4)
        worst = max(worst, err)
    return worst


def test_finite_differences_mlp():
    rng = np.random.default_rng(0)
    net = oracle.Net("mlp", [5, 4, 3])
    X = rng.standard_normal((3, 5)).astype(np.float32)
    y = np.array([0, 2, 1], np.int32)
    assert _fd_check(net, X, y, rng) < 1e-5
    net3 = oracle.Net("mlp", [6, 5, 4, 3])
    X3 = rng.standard_normal((4, 6)).astype(np.float32)
    assert _fd_check(net3, X3, np.array([2, 1, 0, 2], np.int32), rng) < 1e-5


def test_finite_differences_cnn():
    rng = np.random.default_rng(1)
    net = oracle.Net("cnn", [], (6, 6, 2), [(3, 2)], [3])  # LeNet-mini: conv3x3 2->2, pool, fc -> 3
    X = rng.standard_normal((3, 6, 6, 2)).astype(np.float32)
    assert _fd_check(net, X, np.array([0, 1, 2], np.int32), rng) < 1e-5
    net2 = oracle.Net("cnn", [], (12, 12, 2), [(3, 3), (2, 4)], [5, 3])  # two conv stages + 2 fc
    X2 = rng.standard_normal((2, 12, 12, 2)).astype(np.float32)
    assert _fd_check(net2, X2, np.array([1, 2], np.int32), rng) < 1e-5


def test_softmax_regression_closed_form():
    """One layer: grad W = X^T (softmax(XW+b) - Y) / b, grad b = colsum(...) / b."""
    rng = np.random.default_rng(2)
    net = oracle.Net("mlp", [7, 4])
    X = rng.standard_normal((9, 7)).astype(np.float32)
    y = rng.integers(0, 4, 9).astype(np.int32)
    p = rng.standard_normal(oracle.param_count(net))
    g, loss = oracle.batch_grad(net, p, X, y)
    W, bb = p[:28].reshape(7, 4), p[28:]
    Z = X.astype(np.float64) @ W + bb
    Sm = np.exp(Z - Z.max(1, keepdims=True))
    Sm /= Sm.sum(1, keepdims=True)
    Y = np.eye(4)[y]
    np.testing.assert_allclose(g[:28].reshape(7, 4), X.T.astype(np.float64) @ (Sm - Y) / 9, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(g[28:], (Sm - Y).sum(0) / 9, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(loss, -np.log(Sm[np.arange(9), y]).sum(), rtol=1e-13)


def _torch_mlp_grad(net, p, X, y):
    import torch
    ps, off = [], 0
    for l in range(1, len(net.dims)):
        W = torch.tensor(p[off:off + net.dims[l - 1] * net.dims[l]].reshape(net.dims[l - 1], net.dims[l]),
                         dtype=torch.float64, requires_grad=True)
        off += W.numel()
        b = torch.tensor(p[off:off + net.dims[l]], dtype=torch.float64, requires_grad=True)
        off += b.numel()
        ps += [W, b]
    a = torch.tensor(X, dtype=torch.float64)
    for l in range(len(ps) // 2):
        a = a @ ps[2 * l] + ps[2 * l + 1]
        if l < len(ps) // 2 - 1:
            a = torch.relu(a)
    loss = torch.nn.functional.cross_entropy(a, torch.tensor(y, dtype=torch.long), reduction="mean")
    loss.backward()
    return np.concatenate([q.grad.numpy().ravel() for q in ps]), float(loss) * X.shape[0]


def test_mlp_matches_torch_autograd_f64():
    rng = np.random.default_rng(3)
    net = oracle.Net("mlp", [784, 128, 10])
    X, y = S.mnist_like(1, 64)
    p = oracle.init_params(net, 42).astype(np.float64)
    p[np.arange(p.size) % 7 == 3] += 0.01  # non-zero biases too
    g, loss = oracle.batch_grad(net, p, X, y)
    gt, losst = _torch_mlp_grad(net, p, X, y)
    np.testing.assert_allclose(g, gt, rtol=1e-10, atol=1e-13)
    assert abs(loss - losst) < 1e-10 * abs(losst)


def test_cnn_matches_torch_autograd_f64():
    import torch
    F = torch.nn.functional
    net = oracle.Net("cnn", [], (32, 32, 3), [(5, 6), (5, 16)], [120, 84, 10])
    X, y = S.cifar_like(1, 6)
    rng = np.random.default_rng(4)
    p = oracle.init_params(net, 42).astype(np.float64) + rng.standard_normal(62006) * 1e-3
    g, loss = oracle.batch_grad(net, p, X, y)
    tab = oracle.tensor_table(net)
    ts = [torch.tensor(p[o:o + s], dtype=torch.float64, requires_grad=True) for o, s in tab]
    a = torch.tensor(X, dtype=torch.float64).permute(0, 3, 1, 2)  # NHWC -> NCHW
    for c, (k, co) in enumerate([(5, 6), (5, 16)]):
        ci = a.shape[1]
        W = ts[2 * c].view(k, k, ci, co).permute(3, 2, 0, 1)  # [kh][kw][ci][co] -> [co][ci][kh][kw]
        a = F.max_pool2d(F.relu(F.conv2d(a, W, ts[2 * c + 1])), 2)
    a = a.permute(0, 2, 3, 1).reshape(a.shape[0], -1)  # flatten (h, w, c), A7
    dims = [400, 120, 84, 10]
    for f in range(3):
        a = a @ ts[4 + 2 * f].view(dims[f], dims[f + 1]) + ts[5 + 2 * f]
        if f < 2:
            a = F.relu(a)
    lt = F.cross_entropy(a, torch.tensor(y, dtype=torch.long), reduction="mean")
    lt.backward()
    gt = np.concatenate([t.grad.numpy() for t in ts])
    np.testing.assert_allclose(g, gt, rtol=1e-9, atol=1e-12)
    assert abs(loss / 6 - float(lt)) < 1e-12


def test_maxpool_first_max_on_ties():
    """A6: with tied window maxima the gradient goes to the first (row-major) element only."""
    net = oracle.Net("cnn", [], (3, 3, 1), [(2, 1)], [2])  # conv 2x2 -> 2x2 -> pool -> 1x1
    p = np.zeros(oracle.param_count(net))
    p[4] = 1.0  # conv bias 1, conv weights 0 -> all four conv outputs tie at 1
    p[5:7] = [0.5, -0.5]  # fc W
    X = np.zeros((1, 3, 3, 1), np.float32)
    g, _ = oracle.batch_grad(net, p, X, np.array([0], np.int32))
    # d loss / d conv-bias = routed gradient from exactly one (the first) window element
    dlogits = np.exp([0.5, -0.5]) / np.exp([0.5, -0.5]).sum() - [1, 0]
    assert abs(g[4] - (dlogits @ [0.5, -0.5])) < 1e-15


# ----------------------------------------------------------------------------- O9 reduce
def test_fold_worked_values():
    assert oracle.fold(np.array([[1.0], [2.0], [3.0], [4.0]]))[0] == 10.0
    assert oracle.fold(np.array([[1.5], [1.5], [1.5]]))[0] == 4.5


def test_fold_error_bound_and_integer_exactness():
    rng = np.random.default_rng(5)
    for P in range(2, 10):
        g = rng.standard_normal((P, 1024))
        G = oracle.fold(g)
        exact = np.array([math.fsum(g[:, e]) for e in range(1024)])
        u = 2.0 ** -53
        gamma = (P - 1) * u / (1 - (P - 1) * u)
        assert np.all(np.abs(G - exact) <= gamma * np.abs(g).sum(0) + 1e-300)
        gi = rng.integers(-2 ** 40, 2 ** 40, (P, 256)).astype(np.float64)
        assert np.array_equal(oracle.fold(gi), gi.sum(0))
        # left fold order: ((g0 + g1) + g2) ...
        acc = g[0].copy()
        for r in range(1, P):
            acc = acc + g[r]
        assert np.array_equal(acc, G)


# ----------------------------------------------------------------------------- O10-O11 update
def _round_f32(x: Fraction) -> float:
    """Correct IEEE round-to-nearest-even of an exact rational to binary32."""
    if x == 0:
        return 0.0
    sgn = -1 if x < 0 else 1
    a = abs(x)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    e = max(e, -126)
    ulp = Fraction(2) ** (e - 23)
    q = round(a / ulp)  # Fraction.__round__ is round-half-even
    return float(np.float32(sgn * q * ulp))


def test_update_f32_is_correctly_rounded_fma():
    rng = np.random.default_rng(6)
    N = 2000
    G = (rng.standard_normal(N) * 10.0 ** rng.integers(-6, 2, N)).astype(np.float32)
    w0 = rng.standard_normal(N).astype(np.float32)
    v0 = (rng.standard_normal(N) * 1e-3).astype(np.float32)
    for P, lr, mu in [(1, 0.01, 0.9), (2, 0.1, 0.9), (4, 0.01, 0.0), (3, 0.05, 0.5), (8, 0.01, 0.9)]:
        w, v = w0.copy(), v0.copy()
        assert oracle.avg_update(G, w, v, P, lr, mu) == 0
        invP = Fraction(float(np.float32(1.0) / np.float32(P)))
        for e in range(0, N, 7):
            gbar = _round_f32(Fraction(float(G[e])) * invP)
            ve = _round_f32(Fraction(float(np.float32(mu))) * Fraction(float(v0[e])) + Fraction(gbar))
            we = _round_f32(-Fraction(float(np.float32(lr))) * Fraction(ve) + Fraction(float(w0[e])))
            assert float(v[e]) == ve and float(w[e]) == we, (P, e)


def test_update_worked_values():
    w, v = np.array([1.0]), np.array([0.0])
    oracle.avg_update(np.array([1.0]), w, v, 1, 0.1, 0.9)
    assert v[0] == 1.0
    oracle.avg_update(np.array([1.0]), w, v, 1, 0.1, 0.9)
    assert abs(v[0] - 1.9) < 1e-15 and abs(w[0] - 0.71) < 1e-15
    # SGD: lr=0.1, w=[1], g=[10] -> [0] (the fused multiply-add leaves the rounding residue of 0.1)
    w, v = np.array([1.0]), np.array([0.0])
    oracle.avg_update(np.array([10.0]), w, v, 1, 0.1, 0.0)
    assert abs(w[0]) < 1e-16
    # zero gradient leaves w bitwise unchanged
    w32 = np.array([0.123456789, -3.5e-12, 7.0], np.float32)
    before = w32.tobytes()
    oracle.avg_update(np.zeros(3, np.float32), w32, np.zeros(3, np.float32), 4, 0.01, 0.9)
    assert w32.tobytes() == before
    # non-finite detection (A17)
    assert oracle.avg_update(np.array([np.nan, 1.0], np.float32), np.zeros(2, np.float32), np.zeros(2, np.float32),
                             1, 0.1, 0.0) == 1


def test_mean_then_invP_equals_sum_over_B_bitwise():
    """A1: local means x fl(1/P) == sum of local sums / B when B/P, P are powers of two."""
    rng = np.random.default_rng(7)
    net = oracle.Net("mlp", [20, 16, 4])
    X = rng.standard_normal((64, 20)).astype(np.float32)
    y = rng.integers(0, 4, 64).astype(np.int32)
    p = rng.standard_normal(oracle.param_count(net)) * 0.3
    B, P = 64, 4
    means = np.stack([oracle.local_grad(net, p, X, y, B, 0, r, P)[0] for r in range(P)])
    gbar = oracle.fold(means) * (1.0 / P)
    sums = means * (B // P)  # mean x b is exact for b a power of two
    assert np.array_equal(gbar, oracle.fold(sums) / B)


# ----------------------------------------------------------------------------- invariants I1, I2
@pytest.mark.parametrize("P", [2, 4])
def test_dp_gradient_equals_sequential_gradient(P):
    net = oracle.Net("mlp", [784, 128, 10])
    X, y = S.mnist_like(1, 1000)
    p = oracle.init_params(net, 42).astype(np.float64)
    B = 64
    for step in (0, 15):  # 15 wraps around n=1000 (15*64 = 960)
        seq, lseq = oracle.local_grad(net, p, X, y, B, step, 0, 1)
        parts = [oracle.local_grad(net, p, X, y, B, step, r, P) for r in range(P)]
        G = oracle.fold(np.stack([g for g, _ in parts])) * (1.0 / P)
        assert np.abs(G - seq).max() <= 1e-12 * np.abs(seq).max()
        assert abs(sum(l for _, l in parts) - lseq) <= 1e-12 * lseq


def test_dp_training_equals_sequential_training_200_steps():
    """Paper Fig. 6 claim as I1 at f64, SPEC acceptance S:518: 200 steps, rel 1e-6."""
    net = oracle.Net("mlp", [784, 128, 10])
    X, y = S.mnist_like(1, 1000)
    ref, w1, v1 = oracle.train(net, X, y, 64, 1, 200, 0.1, 0.0, 42)
    for P in (2, 4):
        recs, wP, vP = oracle.train(net, X, y, 64, P, 200, 0.1, 0.0, 42)
        for a, b in zip(ref, recs):
            assert abs(a.loss - b.loss) <= 1e-6 * abs(a.loss)
        assert np.abs(wP - w1).max() <= 1e-6 * np.abs(w1).max()
    assert ref[-1].loss < ref[0].loss  # it trains


def test_replicas_bit_identical_and_broadcast_is_needed():
    net = oracle.Net("mlp", [784, 128, 10])
    # without the broadcast, replicas initialised with init_seed + r differ
    assert oracle.init_params(net, 42).tobytes() != oracle.init_params(net, 43).tobytes()
    X, y = S.mnist_like(1, 1000)
    recs, w, v = oracle.train(net, X, y, 64, 4, 5, 0.01, 0.9, 42, check_replicas=True)
    assert len(recs) == 5


def test_cnn_dp_equals_sequential():
    net = oracle.Net("cnn", [], (32, 32, 3), [(5, 6), (5, 16)], [120, 84, 10])
    X, y = S.cifar_like(1, 64)
    p = oracle.init_params(net, 42).astype(np.float64)
    seq, _ = oracle.local_grad(net, p, X, y, 16, 1, 0, 1)
    G = oracle.fold(np.stack([oracle.local_grad(net, p, X, y, 16, 1, r, 4)[0] for r in range(4)])) * 0.25
    assert np.abs(G - seq).max() <= 1e-12 * np.abs(seq).max()


# ----------------------------------------------------------------------------- tf32emu (readings A12 / A23)
def test_tf32_truncation_measured_values_and_properties():
    """A12: the values tools/tc_probe.cu measured on B200 (1+2^-11+2^-12 -> 1, 1+3*2^-11 -> 1+2^-10), and
    what truncation of the low 13 mantissa bits implies: sign symmetry, |tf32(x)| <= |x| with relative
    gap < 2^-10, TF32-representable values fixed, fp32 rounding first."""
    assert oracle.tf32(1 + 2**-11 + 2**-12) == 1.0
    assert oracle.tf32(1 + 3 * 2**-11) == 1 + 2**-10
    rng = np.random.default_rng(12)
    for x in rng.standard_normal(2000) * 10.0 ** rng.integers(-6, 6, 2000):
        t = oracle.tf32(x)
        assert oracle.tf32(-x) == -t
        x32 = float(np.float32(x))
        assert abs(t) <= abs(x32) and abs(x32 - t) < 2**-10 * abs(x32)
        assert oracle.tf32(t) == t
        m = np.frexp(t)[0] * 2**11  # 11 significant bits (1 implicit + 10 stored)
        assert m == int(m)
    assert oracle.tf32(1 + 2**-10) == 1 + 2**-10  # exactly representable: unchanged
    assert oracle.tf32(1 + 2**-30) == 1.0          # rounds to fp32 1.0 first


def test_tf32emu_is_exact_when_no_contraction_is_tensor_core_shaped():
    """Widths < 16 (A23: CUDA-core fp32 contractions) -> tf32emu is the f64 oracle, bitwise."""
    net = oracle.Net("mlp", [12, 8, 3])
    X = np.random.default_rng(4).standard_normal((16, 12)).astype(np.float32)
    y = (np.arange(16) % 3).astype(np.int32)
    p = oracle.init_params(net, 5).astype(np.float64)
    g0, l0 = oracle.local_grad(net, p, X, y, 16, 0, 0, 1)
    g1, l1 = oracle.local_grad(net, p, X, y, 16, 0, 0, 1, tf32emu=True)
    assert np.array_equal(g0, g1) and l0 == l1


def test_tf32emu_is_exact_on_tf32_representable_operands():
    """[8, 16, 3]: only layer 1's forward is tensor-core shaped (d_1 = 16 >= 16; its weight gradient needs
    d_1 > 16; the head is fp32).  With X and W_1 holding values of <= 11 significant bits the truncation is
    the identity, so tf32emu equals the f64 oracle bitwise -- truncation touches operands only."""
    net = oracle.Net("mlp", [8, 16, 3])
    rng = np.random.default_rng(6)
    X = (rng.integers(-64, 64, (32, 8)) / 32.0).astype(np.float32)
    y = (np.arange(32) % 3).astype(np.int32)
    p = oracle.init_params(net, 7).astype(np.float64)
    (o_w1, n_w1), = oracle.tensor_table(net)[:1]
    p[o_w1:o_w1 + n_w1] = rng.integers(-512, 512, n_w1) / 1024.0
    g0, l0 = oracle.local_grad(net, p, X, y, 32, 0, 0, 1)
    g1, l1 = oracle.local_grad(net, p, X, y, 32, 0, 0, 1, tf32emu=True)
    assert np.array_equal(g0, g1) and l0 == l1
    p[o_w1] += 2**-13  # one weight no longer TF32-representable: the emulation now differs
    g0, _ = oracle.local_grad(net, p, X, y, 32, 0, 0, 1)
    g1, _ = oracle.local_grad(net, p, X, y, 32, 0, 0, 1, tf32emu=True)
    assert not np.array_equal(g0, g1)


def test_tf32emu_forward_truncates_toward_zero_within_bound():
    """Non-negative inputs and weights: truncating both operands toward zero can only lower each product,
    by < (2^-9 + 2^-20) of it (two 2^-10 relative gaps), so 0 <= exact - emu <= (2^-9 + 2^-20) * exact
    for the pre-activations (biases zero) -- and the gap is not zero."""
    net = oracle.Net("mlp", [32, 64, 3])
    rng = np.random.default_rng(8)
    X = rng.random((20, 32)).astype(np.float32)
    y = (np.arange(20) % 3).astype(np.int32)
    p = np.abs(oracle.init_params(net, 9).astype(np.float64))
    (o_b1, n_b1) = oracle.tensor_table(net)[1]
    p[o_b1:o_b1 + n_b1] = 0.0
    ex = oracle.mlp_activations(net, p, X, y, 1)
    em = oracle.mlp_activations(net, p, X, y, 1, tf32emu=True)
    gap = ex - em
    assert (gap >= 0).all() and (gap <= (2**-9 + 2**-20) * ex + 1e-300).all()
    assert gap.max() > 0
