"""Run-to-run bitwise determinism of every path with hand-rolled synchronisation (compute-sanitizer is closed
on this pool, profiles/round2_sanitizer.md): split-K tickets and DSMEM cluster folds, CTA-pair barriers,
the double-buffered TMEM / shared-memory pipeline of the tensor-core convolutions, the fused head's
ordered loss fold, and the simulated-rank fused NVLink protocol.  Each is repeated from fresh contexts and
must give bitwise-identical results (a race shows up as a difference); the values themselves are checked
against the oracle by the parity tests."""
from __future__ import annotations

import numpy as np
import pytest

import mtx_synth as S

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1704_04560_b200 as P  # noqa: E402
from paper_1704_04560_b200 import mtx  # noqa: E402

TC = "tcgen05" in mtx.mtx_build_info()
PRECS = [P.MTX_FP32] + ([P.MTX_3XTF32, P.MTX_3XF16] if TC else [])


def _trajectory(cfg, X, y, prec, steps):
    r = P.Replica(cfg, precision=prec)
    try:
        r.bcast()
        r.shard(X, y)
        losses = [r.step(want_loss=True) for _ in range(steps)]
        return losses, r.get().tobytes(), r.get(P.MTX_BUF_VELOCITY).tobytes(), r.get(P.MTX_BUF_GRADS).tobytes()
    finally:
        r.close()


@pytest.mark.parametrize("prec", PRECS)
@pytest.mark.parametrize("name", ["cfg4", "cfg3"])
def test_step_bitwise_repeatable(name, prec):
    """Full-size launch configurations (cfg4 B = 8192: pair / cluster split-K GEMMs, head with > 2048 rows;
    cfg3 B = 1024: the tensor-core convolutions' persistent pipeline), 3 steps, 3 fresh contexts."""
    if name == "cfg4":
        cfg = dict(S.CONFIGS["cfg4"], n=20000)
        X, y = S.higgs_like(1, 20000)
    else:
        cfg = dict(S.CONFIGS["cfg3"], n=2048)
        X, y = S.cifar_like(1, 2048)
    runs = [_trajectory(cfg, X, y, prec, 3) for _ in range(3)]
    for r in runs[1:]:
        assert r == runs[0]


@pytest.mark.skipif(not TC, reason="tcgen05 engine not built")
@pytest.mark.parametrize("shape", [(8192, 1024, 1024, 0, 0, 1), (8192, 1024, 1024, 0, 1, 3), (1024, 1024, 8192, 1, 0, 0),
                                   (784, 512, 512, 1, 0, 0), (512, 512, 784, 0, 0, 1), (28, 1024, 8192, 1, 0, 0)])
@pytest.mark.parametrize("engine", [2, 4])
def test_gemm_bitwise_repeatable(shape, engine):
    M, N, K, ta, tb, epi = shape
    rng = np.random.default_rng(M + N + K)
    A = torch.from_numpy(rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)).cuda()
    B = torch.from_numpy(rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)).cuda()
    bias = torch.from_numpy(rng.standard_normal(N).astype(np.float32)).cuda()
    mask = torch.from_numpy(np.maximum(rng.standard_normal((M, N)), 0).astype(np.float32)).cuda()
    outs = []
    for _ in range(3):
        r = P.Replica(dict(S.CONFIGS["cfg4"], B=1024), precision=P.MTX_3XTF32 if engine == 2 else P.MTX_3XF16)
        try:
            C = torch.full((M, N), np.nan, device="cuda")
            torch.cuda.synchronize()
            for _ in range(2):  # the second call reuses the first one's split-K tickets / scratch
                mtx.mtx_debug_gemm(r.ctx, engine, M, N, K, ta, tb, epi, A.data_ptr(), M if ta else K, B.data_ptr(),
                                   K if tb else N, C.data_ptr(), N, bias.data_ptr(), mask.data_ptr(), N, r.s)
            r.sync()
            outs.append(C.cpu().numpy().tobytes())
        finally:
            r.close()
    assert outs[1] == outs[0] and outs[2] == outs[0]


@pytest.mark.parametrize("proto", ["pull", "push"])
def test_fused_protocol_bitwise_repeatable(proto):
    mode = P.MTX_REDUCE_FUSED | (P.MTX_DEBUG_REDUCE_PUSH if proto == "push" else 0)
    n, Pn = (1 << 20) + 4, 8
    g = np.zeros((Pn, n + 32), np.float32)
    for q in range(Pn):
        g[q, :n] = S.cfg5_grad_random(2, q, n)
    w, v = S.cfg5_params(2, n), S.cfg5_velocity(2, n)
    outs = []
    for _ in range(3):
        r = P.Replica(dict(S.CONFIGS["cfg1"], B=4))
        try:
            dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
            gd, wd, vd = [dev(g[q]) for q in range(Pn)], [dev(w) for _ in range(Pn)], [dev(v) for _ in range(Pn)]
            Gd = [torch.zeros(n + 32, device="cuda") for _ in range(Pn)]
            torch.cuda.synchronize()
            mtx.mtx_debug_reduce(r.ctx, mode, Pn, [t.data_ptr() for t in gd], [t.data_ptr() for t in wd],
                                 [t.data_ptr() for t in vd], [t.data_ptr() for t in Gd], n, 0.01, 0.9, r.s)
            r.sync()
            r.get()
            outs.append(b"".join(t.cpu().numpy().tobytes() for t in wd + vd + Gd))
        finally:
            r.close()
    assert outs[1] == outs[0] and outs[2] == outs[0]
