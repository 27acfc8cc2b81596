"""P > 1 reduction arithmetic on ONE GPU (the driver's round-end box has one): mtx_debug_reduce runs the
product kernels of the multi-GPU modes for P simulated ranks whose buffers all live on this device --
FUSED with its real cross-rank flag-barrier protocol on P concurrent streams, ORDERED with its gather +
ascending-rank fold -- and both must equal the oracle's fp32 left fold (O9, reading A2), x fl(1/P) (O10,
A3) and momentum update (O11, A4) BIT-EXACTLY on random (non-dyadic) gradients, for P = 2, 4 and 8
(SURVEY.md §8(c) O9-O11).  P = 8 is a world no gpurun box offers."""
from __future__ import annotations

import numpy as np
import pytest

import mtx_synth as S
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1704_04560_b200 as P  # noqa: E402
from paper_1704_04560_b200 import mtx  # noqa: E402

LOSS_SLOT = 32
ALEXNET = 61_100_840  # SURVEY.md §8(a) cfg5 AlexNet point


@pytest.fixture(scope="module")
def rep():
    r = P.Replica(dict(S.CONFIGS["cfg1"], B=4))
    yield r
    r.close()


def _inputs(P_, n, seed=1):
    g = np.zeros((P_, n + LOSS_SLOT), np.float32)
    for q in range(P_):
        g[q, :n] = S.cfg5_grad_random(seed, q, n)
        g[q, n] = np.float32(1.0 + 0.37 * q)  # this rank's local loss sum
    return g, S.cfg5_params(seed, n), S.cfg5_velocity(seed, n)


def _slice(n, P_, r):
    n4 = n // 4
    return 4 * (n4 * r // P_), 4 * (n4 * (r + 1) // P_)


def _run(rep, mode, P_, g, w, v, mu, lr=0.01):
    n = w.size
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    gd = [dev(g[q]) for q in range(P_)]
    Gd = [torch.full((n + LOSS_SLOT,), np.nan, device="cuda") for _ in range(P_)]
    wd = [dev(w) for _ in range(P_)]  # replicas after the broadcast: identical w
    vd = [dev(v) for _ in range(P_)] if mu else None
    torch.cuda.synchronize()
    mtx.mtx_debug_reduce(rep.ctx, mode, P_, [t.data_ptr() for t in gd], [t.data_ptr() for t in wd],
                         [t.data_ptr() for t in vd] if mu else None, [t.data_ptr() for t in Gd], n, lr, mu, rep.s)
    rep.sync()
    return Gd, wd, vd


def same(dev_t, ref: np.ndarray) -> bool:
    """Bitwise equality of a device result with an oracle array (compared on the device: no host copies
    of the P replicas at the AlexNet size)."""
    r = torch.from_numpy(np.ascontiguousarray(ref, np.float32)).cuda()
    return bool(torch.equal(dev_t.view(torch.int32), r.view(torch.int32)))


def _oracle(g, w, v, P_, mu, lr=0.01):
    n = w.size
    G = oracle.fold(g)  # f32 ascending-rank left fold over [P, n + loss slot]
    wo, vo = w.copy(), (v.copy() if mu else np.zeros_like(w))
    oracle.avg_update(G[:n].copy(), wo, vo, P_, lr, mu)
    return G, wo, vo


FUSED_MODES = {"pull": P.MTX_REDUCE_FUSED, "push": P.MTX_REDUCE_FUSED | P.MTX_DEBUG_REDUCE_PUSH}


@pytest.mark.parametrize("proto", ["pull", "push"])
@pytest.mark.parametrize("P_", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1000, (1 << 20) + 4])
@pytest.mark.parametrize("mu", [0.9, 0.0])
def test_fused_protocol_bit_exact(rep, P_, n, mu, proto):
    """MTX_REDUCE_FUSED, both protocols (pull: the kernel loads the peers' g over NVLink; push: the peers' copy
    engines wrote them into the owner's landing area -- unequal shares when P does not divide n / 4): every
    replica's w equals the oracle's everywhere; each owner's slice of v and G equals the oracle's; the loss slot
    is the rank-ordered fold on every rank."""
    g, w, v = _inputs(P_, n)
    Gs, ws, vs = _run(rep, FUSED_MODES[proto], P_, g, w, v, mu)
    G, wo, vo = _oracle(g, w, v, P_, mu)
    for q in range(P_):
        assert same(ws[q], wo), f"replica {q} w"
        lo, hi = _slice(n, P_, q)
        assert same(Gs[q][lo:hi], G[lo:hi]), f"owner {q} G slice"
        if mu:
            assert same(vs[q][lo:hi], vo[lo:hi]), f"owner {q} v slice"
        assert same(Gs[q][n + 1:n + 2], G[n:n + 1]), f"rank {q} folded loss"


@pytest.mark.parametrize("P_", [2, 4, 8])
@pytest.mark.parametrize("n", [1000, (1 << 20) + 4])
def test_ordered_fold_and_update_bit_exact(rep, P_, n):
    """MTX_REDUCE_ORDERED: gather + ascending-rank fold on every rank, then avg_update with fl(1/P)."""
    g, w, v = _inputs(P_, n, seed=3)
    Gs, ws, vs = _run(rep, P.MTX_REDUCE_ORDERED, P_, g, w, v, 0.9)
    G, wo, vo = _oracle(g, w, v, P_, 0.9)
    for r in range(P_):
        assert same(Gs[r][:n + 1], G[:n + 1]), f"rank {r} G"
        assert same(ws[r], wo), f"rank {r} w"
        assert same(vs[r], vo), f"rank {r} v"


@pytest.mark.parametrize("proto", ["pull", "push"])
def test_fused_protocol_alexnet_size_p8(rep, proto):
    """The AlexNet-scale flat buffer (61.1 M parameters) at P = 8, momentum."""
    n = ALEXNET
    P_ = 8
    g, w, v = _inputs(P_, n, seed=5)
    Gs, ws, vs = _run(rep, FUSED_MODES[proto], P_, g, w, v, 0.9)
    G, wo, vo = _oracle(g, w, v, P_, 0.9)
    for q in range(P_):
        assert same(ws[q], wo), f"replica {q} w"
        lo, hi = _slice(n, P_, q)
        assert same(Gs[q][lo:hi], G[lo:hi])
        assert same(vs[q][lo:hi], vo[lo:hi])


def test_fused_protocol_flags_non_finite():
    """A NaN in one simulated rank's gradient reaches every average it enters: MTX_ERR_NUMERIC (A17)."""
    r = P.Replica(dict(S.CONFIGS["cfg1"], B=4))
    try:
        g, w, v = _inputs(4, 4096, seed=7)
        g[2, 1234] = np.nan
        _run(r, P.MTX_REDUCE_FUSED, 4, g, w, v, 0.9)
        with pytest.raises(P.MtxError) as e:
            r.get()
        assert e.value.status == 6
    finally:
        r.close()


def test_nccl_modes_are_not_simulated(rep):
    with pytest.raises(P.MtxError) as e:
        g, w, v = _inputs(2, 64)
        _run(rep, P.MTX_REDUCE_NCCL, 2, g, w, v, 0.9)
    assert e.value.status == 9
