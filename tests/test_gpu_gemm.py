"""Kernel-level parity of the local contractions (both engines) against the
definition C = op(A) op(B) (+ epilogue) computed in float64 by numpy, for the
three layouts the step issues: forward (A, B row-major), dgrad (B transposed)
and wgrad (A transposed), with ragged edges and several tiles."""
from __future__ import annotations

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import mtx_synth as S  # noqa: E402
import paper_1704_04560_b200 as P  # noqa: E402
from paper_1704_04560_b200 import mtx  # noqa: E402
from tests._util import maxrel  # noqa: E402

TC = "tcgen05" in mtx.mtx_build_info()


@pytest.fixture(scope="module")
def rep():
    r = P.Replica(dict(S.CONFIGS["cfg4"], B=1024), precision=P.MTX_3XTF32 if TC else P.MTX_FP32)
    yield r
    r.close()


SHAPES = [  # (M, N, K) incl. the step's shapes: cfg4 fwd/dgrad/wgrad, cfg2, K = 28, ragged M/N/K
    (1024, 1024, 1024), (512, 512, 784), (8192, 1024, 28), (28, 1024, 2048), (300, 200, 100), (128, 64, 96),
    (1000, 384, 520), (1024, 640, 256), (64, 784, 512),  # tcgen05 N-tile 64 / 32 plans
    (4096, 1024, 256), (4000, 512, 200),  # CTA-pair (cta_group::2) 256 x 128 tiles, ragged M / K
    (8192, 1024, 256), (8100, 640, 300),  # stream-K remainder (last round split into K-halves), ragged
    (8192, 1024, 1024), (8000, 1024, 1000),  # 3xTF32 CTA-pair 256 x 256 tiles (N = 256 MMAs), ragged M / K
    (1024, 1024, 8192), (768, 512, 4000),  # ... and their split-K weight-gradient plan, ragged K
]


def _run(rep, engine, M, N, K, ta, tb, epi, rng):
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    mask = np.maximum(rng.standard_normal((M, N)), 0).astype(np.float32)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    Ad, Bd, bd, md = d(A), d(B), d(bias), d(mask)
    Cd = torch.full((M, N), np.nan, device="cuda")
    torch.cuda.synchronize()
    mtx.mtx_debug_gemm(rep.ctx, engine, M, N, K, ta, tb, epi, Ad.data_ptr(), M if ta else K, Bd.data_ptr(),
                       K if tb else N, Cd.data_ptr(), N, bd.data_ptr(), md.data_ptr(), N, rep.s)
    rep.sync()
    a = A.T.astype(np.float64) if ta else A.astype(np.float64)
    b = B.T.astype(np.float64) if tb else B.astype(np.float64)
    ref = a @ b
    if epi == 1:
        ref = np.maximum(ref + bias, 0)
    elif epi == 2:
        ref = ref + bias
    elif epi == 3:
        ref = np.where(mask > 0, ref, 0)
    return Cd.cpu().numpy(), ref


@pytest.mark.parametrize("engine", [0, 2] if TC else [0])
@pytest.mark.parametrize("layout", [(0, 0, 1), (0, 0, 2), (0, 1, 3), (1, 0, 0)])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_layouts(rep, engine, layout, shape):
    ta, tb, epi = layout
    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    try:
        C, ref = _run(rep, engine, M, N, K, ta, tb, epi, rng)
    except P.MtxError:
        raise
    assert not np.isnan(C).any()
    # fp32 tier (SIMT, 3xTF32): fp32 products and sums
    assert maxrel(C, ref) <= 1e-5 * max(1.0, np.sqrt(K / 1024)), maxrel(C, ref)


@pytest.fixture(scope="module")
def rep16():
    r = P.Replica(dict(S.CONFIGS["cfg4"], B=1024), precision=P.MTX_3XF16)
    yield r
    r.close()


@pytest.mark.skipif(not TC, reason="tcgen05 engine not built")
@pytest.mark.parametrize("layout", [(0, 0, 1), (0, 0, 2), (0, 1, 3), (1, 0, 0)])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_layouts_3xf16(rep16, layout, shape):
    """3xF16 engine (diagnostic engine 4: A and B quantized to fp16 hi/lo planes with one power-of-two
    scale per operand, then kind::f16 MMAs): the fp32 tier against the float64 definition."""
    ta, tb, epi = layout
    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    C, ref = _run(rep16, 4, M, N, K, ta, tb, epi, rng)
    assert not np.isnan(C).any()
    assert maxrel(C, ref) <= 1e-5 * max(1.0, np.sqrt(K / 1024)), maxrel(C, ref)


@pytest.mark.skipif(not TC, reason="tcgen05 engine not built")
@pytest.mark.parametrize("scales", [(1e-7, 3e4), (2.0 ** 40, 2.0 ** -60), (1e-20, 1e-8)])
def test_gemm_3xf16_exponent_range(rep16, scales):
    """The per-tensor power-of-two scale carries operands far outside fp16's range (|x| up to 2^40, down to
    1e-20) through the fp16 planes: the result keeps the fp32 tier."""
    M, N, K = 1000, 384, 520
    rng = np.random.default_rng(7)
    sa, sb = scales
    A = (rng.standard_normal((M, K)) * sa).astype(np.float32)
    B = (rng.standard_normal((K, N)) * sb).astype(np.float32)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    Ad, Bd = d(A), d(B)
    Cd = torch.full((M, N), np.nan, device="cuda")
    torch.cuda.synchronize()
    mtx.mtx_debug_gemm(rep16.ctx, 4, M, N, K, 0, 0, 0, Ad.data_ptr(), K, Bd.data_ptr(), N, Cd.data_ptr(), N,
                       None, None, 0, rep16.s)
    rep16.sync()
    ref = A.astype(np.float64) @ B.astype(np.float64)
    assert maxrel(Cd.cpu().numpy(), ref) <= 1e-5


def _tf32_trunc(x: np.ndarray) -> np.ndarray:
    """fp32 -> TF32 by truncating the low 13 mantissa bits: how tcgen05 kind::tf32 consumes fp32
    shared-memory operands (reading A12, measured with tools/tc_probe.cu)."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)


@pytest.mark.skipif(not TC, reason="tcgen05 engine not built")
@pytest.mark.parametrize("layout", [(0, 0, 1), (0, 1, 3), (1, 0, 0)])
@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (512, 512, 784), (1024, 640, 256), (8192, 1024, 28),
                                   (4000, 512, 200), (8100, 640, 300)])
def test_tf32_hardware_truncation_reading_a12(rep, layout, shape):
    """Pins reading A12 (how tcgen05 kind::tf32 consumes fp32 shared-memory operands), not a product
    precision: the raw one-MMA-per-k-step contraction (diagnostic engine 1; 1xTF32 is not a product
    mode, A22) equals both operands truncated to TF32 with exact products and fp32
    accumulation.  The 3xTF32 planes are TF32-representable, so they pass through this rule exactly."""
    ta, tb, epi = layout
    M, N, K = shape
    rng = np.random.default_rng(M + 5 * N + 11 * K)
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    bias = rng.standard_normal(N).astype(np.float32)
    mask = np.maximum(rng.standard_normal((M, N)), 0).astype(np.float32)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    Ad, Bd, bd, md = d(A), d(B), d(bias), d(mask)
    Cd = torch.full((M, N), np.nan, device="cuda")
    torch.cuda.synchronize()
    mtx.mtx_debug_gemm(rep.ctx, 1, M, N, K, ta, tb, epi, Ad.data_ptr(), M if ta else K, Bd.data_ptr(),
                       K if tb else N, Cd.data_ptr(), N, bd.data_ptr(), md.data_ptr(), N, rep.s)
    rep.sync()
    a = _tf32_trunc(A.T if ta else A).astype(np.float64)
    b = _tf32_trunc(B.T if tb else B).astype(np.float64)
    ref = a @ b
    if epi == 1:
        ref = np.maximum(ref + bias, 0)
    elif epi == 3:
        ref = np.where(mask > 0, ref, 0)
    C = Cd.cpu().numpy()
    exact = (A.T if ta else A).astype(np.float64) @ (B.T if tb else B).astype(np.float64)
    if epi == 1:
        exact = np.maximum(exact + bias, 0)
    elif epi == 3:
        exact = np.where(mask > 0, exact, 0)
    e_emu, e_exact = maxrel(C, ref), maxrel(C, exact)
    # fp32 accumulation of K products: <= ~K * 2^-24 worst case, ~sqrt(K) * 2^-24 typical
    assert e_emu <= 2e-6 * max(1.0, np.sqrt(K / 256)), (e_emu, e_exact)
    assert e_emu < e_exact / 20, (e_emu, e_exact)  # the emulation explains the TF32 error
