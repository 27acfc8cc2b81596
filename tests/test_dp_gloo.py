"""World-size-2 multi-process test of the data-parallel host logic on CPU (gloo):
the Global Broadcast of the initial variables, each rank's contiguous slice of the
global batch (mtx_batch_slice from libmtx, a pure host function), local gradients
on the slice (oracle), an allreduce-sum through torch.distributed and x 1/P --
which must equal the sequential full-batch gradient."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    import mtx_synth as S
    import oracle
    from paper_1704_04560_b200 import mtx
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        net = oracle.Net("mlp", [784, 64, 10])
        X, y = S.mnist_like(1, 300)
        B = 32
        w = torch.from_numpy(oracle.init_params(net, 42 + rank).astype(np.float64))
        dist.broadcast(w, src=0)  # Global Broadcast
        assert np.array_equal(w.numpy(), oracle.init_params(net, 42).astype(np.float64))
        for step in (0, 9):  # 9*32 = 288: the window wraps around n = 300
            (b0, b1), (l0, l1) = mtx.mtx_batch_slice(300, B, step, rank, world)
            rows = np.r_[b0:b0 + l0, b1:b1 + l1]
            assert len(rows) == B // world
            g, lsum = oracle.batch_grad(net, w.numpy(), X[rows], y[rows])
            gt = torch.from_numpy(g)
            lt = torch.tensor([lsum], dtype=torch.float64)
            dist.all_reduce(gt)
            dist.all_reduce(lt)
            gbar = gt.numpy() * (1.0 / world)
            seq, lseq = oracle.local_grad(net, w.numpy(), X, y, B, step, 0, 1)
            assert np.abs(gbar - seq).max() <= 1e-12 * np.abs(seq).max()
            assert abs(float(lt[0]) - lseq) <= 1e-12 * lseq
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback
        q.put((rank, traceback.format_exc() + str(e)))


def test_two_rank_gloo_dp_equals_sequential():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(60)
    assert res == {0: "ok", 1: "ok"}, res
