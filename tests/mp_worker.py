"""Multi-rank GPU parity worker, launched by tests/test_multigpu.py under torchrun
(one process per GPU, NCCL data path, gloo for the uid and result exchange).

Checks, per rank, against the oracle's DP(P) simulation:
  * Global Broadcast: before it, replicas initialised with init_seed + r differ
    (negative control); after it, every rank's parameters are bitwise rank
    0's oracle init.
  * Replica identity I2: the parameter/velocity digest is equal on all ranks after
    every step.
  * I1 across implementations: GPU DP(P) losses and weights vs oracle DP(P) within
    the tier tolerance; the reduced gradient G vs the oracle's fold.
  * The averaging operator on dyadic gradients is bit-exact vs the oracle (any
    summation order is exact on those inputs, A2).
  * MTX_REDUCE_ORDERED reproduces the NCCL result bitwise at P = 2 (addition commutes).
"""
from __future__ import annotations

import json
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import mtx_synth as S  # noqa: E402
import oracle  # noqa: E402
import paper_1704_04560_b200 as P  # noqa: E402
from paper_1704_04560_b200 import mtx  # noqa: E402
from tests._parity import step_errors  # noqa: E402
from tests._util import GRAD_TOL, TOL, maxrel  # noqa: E402


def allgather_obj(x):
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, x)
    return out


def check(cond, msg):
    if not cond:
        raise AssertionError(msg)


def run_model(rank, world, cfg, X, y, steps, precision, reduce=P.MTX_REDUCE_NCCL, bucket=256 << 10):
    uid = P.nccl_uid_broadcast(rank, world)
    r = P.Replica(cfg, rank=rank, world=world, uid=uid, device=rank, precision=precision, reduce=reduce,
                  bucket_bytes=bucket)
    try:
        d0 = allgather_obj(r.digest())
        check(len(set(d0)) == world, "replicas should differ before the broadcast (distinct init seeds)")
        r.bcast()
        net = oracle.Net.from_cfg(cfg)
        w0 = r.get()
        check(np.array_equal(w0.view(np.uint32), oracle.init_params(net, 42).view(np.uint32)),
              f"rank {rank}: params after broadcast != oracle rank-0 init")
        r.shard(X, y)
        out = []
        for t in range(steps):
            loss = r.step(want_loss=True)
            dg = allgather_obj(r.digest())
            check(len(set(dg)) == 1, f"step {t}: replica digests differ {dg}")
            out.append((loss, r.get(P.MTX_BUF_GRADS), r.get(P.MTX_BUF_PARAMS), r.get(P.MTX_BUF_VELOCITY)))
            dist.barrier()  # every rank has read its state before any rank starts the next step
        return out
    finally:
        r.close()


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    report = {"rank": rank, "world": world, "checks": []}
    try:
        # ---- averaging operator on dyadic gradients: bit-exact vs oracle fold + update
        cfg_tiny = dict(S.CONFIGS["cfg1"], B=4 * world)
        uid = P.nccl_uid_broadcast(rank, world)
        r = P.Replica(cfg_tiny, rank=rank, world=world, uid=uid, device=rank)
        for n in (1000, (1 << 20) + 3, 61_100_840 // 16):
            g_all = np.stack([S.cfg5_grad_dyadic(1, q, n) for q in range(world)])
            w = S.cfg5_params(1, n)
            v = S.cfg5_velocity(1, n)
            Gd = torch.from_numpy(g_all[rank].copy()).cuda()
            wd = torch.from_numpy(w.copy()).cuda()
            vd = torch.from_numpy(v.copy()).cuda()
            torch.cuda.synchronize()
            mtx.mtx_allreduce_avg(r.ctx, Gd.data_ptr(), wd.data_ptr(), vd.data_ptr(), n, 0.01, 0.9, 1, r.s)
            r.sync()
            G = oracle.fold(g_all)
            wo, vo = w.copy(), v.copy()
            oracle.avg_update(G, wo, vo, world, 0.01, 0.9)
            check(np.array_equal(Gd.cpu().numpy().view(np.uint32), G.view(np.uint32)), f"allreduce n={n}")
            check(np.array_equal(wd.cpu().numpy().view(np.uint32), wo.view(np.uint32)), f"update w n={n}")
            check(np.array_equal(vd.cpu().numpy().view(np.uint32), vo.view(np.uint32)), f"update v n={n}")
        r.close()
        report["checks"].append("allreduce_avg dyadic bit-exact")

        # ---- the training step, DP(P) vs oracle DP(P)
        precisions = [P.MTX_FP32] + ([P.MTX_3XTF32, P.MTX_3XF16] if "tcgen05" in mtx.mtx_build_info() else [])
        for prec in precisions:
            tol, gtol = TOL[prec], GRAD_TOL[prec]
            runs = [("cfg1", 64, 5), ("cfg2", 512, 3), ("cfg3", 64, 2)]
            if prec == P.MTX_3XF16:  # cfg4's shape: the 28-feature CUDA-core forward, lean outputs, fused maxima
                runs.append(("cfg4", 512, 2))
            for name, B, steps in runs:
                cfg = dict(S.CONFIGS[name], B=B)
                if name == "cfg3":
                    X, y = S.cifar_like(1, 300)
                elif name == "cfg4":
                    X, y = S.higgs_like(1, 2048)
                else:
                    X, y = S.mnist_like(1, 1000 if name == "cfg1" else 4096)
                gpu = run_model(rank, world, cfg, X, y, steps, prec)
                recs, w_ref, _ = oracle.train(oracle.Net.from_cfg(cfg), X, y, B, world, steps, cfg["lr"], cfg["mu"],
                                              42, keep_grads=True)
                net = oracle.Net.from_cfg(cfg)
                w0 = oracle.init_params(net, 42)
                v0 = np.zeros_like(w0)
                for t, (rec, g) in enumerate(zip(recs, gpu)):
                    check(abs(g[0] - rec.loss) <= tol * abs(rec.loss), f"{name} step {t} loss {g[0]} vs {rec.loss}")
                    e = step_errors(net, cfg, X, y, t, w0, v0, g, world)
                    check(max(e.values()) <= gtol, f"{name} step {t} errors {e}")
                    w0, v0 = g[2], g[3]
                e = maxrel(gpu[-1][2], w_ref)
                check(e <= gtol, f"{name} weights err {e}")
                report["checks"].append(f"{name} DP({world}) prec={prec} vs oracle ok")
        # ---- the averaging operator on arbitrary fp32 gradients (mtx_sync_update): ORDERED and FUSED are
        #      bit-exact with the oracle's f32 left fold + update; NCCL within the gamma_{P-1} bound
        cfg = dict(S.CONFIGS["cfg2"], B=64 * world)
        net = oracle.Net.from_cfg(cfg)
        N = oracle.param_count(net)
        rng = np.random.default_rng(123)
        g_all = (rng.standard_normal((world, N)) * 10.0 ** rng.integers(-6, 0, (world, N))).astype(np.float32)
        w0 = oracle.init_params(net, 42)
        v0 = (rng.standard_normal(N) * 1e-3).astype(np.float32)
        Gref = oracle.fold(g_all)
        wref, vref = w0.copy(), v0.copy()
        oracle.avg_update(Gref, wref, vref, world, cfg["lr"], cfg["mu"])
        for mode in (P.MTX_REDUCE_ORDERED, P.MTX_REDUCE_FUSED, P.MTX_REDUCE_NCCL, P.MTX_REDUCE_LAYERWISE,
                     P.MTX_REDUCE_ZERO1):
            uid = P.nccl_uid_broadcast(rank, world)
            r = P.Replica(cfg, rank=rank, world=world, uid=uid, device=rank, reduce=mode, bucket_bytes=1 << 20)
            r.bcast()
            r.set(P.MTX_BUF_PARAMS, w0)
            r.set(P.MTX_BUF_VELOCITY, v0)
            r.set(P.MTX_BUF_GRADS, g_all[rank])
            mtx.mtx_sync_update(r.ctx, r.s)
            G, wv, vv = r.get(P.MTX_BUF_GRADS), r.get(P.MTX_BUF_PARAMS), r.get(P.MTX_BUF_VELOCITY)
            r.close()
            if mode in (P.MTX_REDUCE_ORDERED, P.MTX_REDUCE_FUSED) or world == 2:
                check(np.array_equal(G.view(np.uint32), Gref.view(np.uint32)), f"sync_update G mode {mode}")
                check(np.array_equal(wv.view(np.uint32), wref.view(np.uint32)), f"sync_update w mode {mode}")
                check(np.array_equal(vv.view(np.uint32), vref.view(np.uint32)), f"sync_update v mode {mode}")
            else:
                u = 2.0 ** -24
                # both NCCL's order and the fold are within gamma_{P-1} sum|g| of the exact sum
                bound = 2 * (world - 1) * u / (1 - (world - 1) * u) * np.abs(g_all.astype(np.float64)).sum(0)
                check(np.all(np.abs(G.astype(np.float64) - Gref) <= bound + 1e-38), "NCCL G outside gamma bound")
        report["checks"].append(f"sync_update ORDERED/FUSED bit-exact vs oracle fold at P={world}; NCCL/LAYERWISE/ZERO1 "
                                "bit-exact at P=2, within gamma bound otherwise")
        # ---- the training step in LAYERWISE and ZERO1 modes (replica digests checked every step)
        cfg = dict(S.CONFIGS["cfg2"], B=512)
        X, y = S.mnist_like(1, 4096)
        recs, w_ref, _ = oracle.train(oracle.Net.from_cfg(cfg), X, y, 512, world, 2, cfg["lr"], cfg["mu"], 42,
                                      keep_grads=True)
        for mode in (P.MTX_REDUCE_LAYERWISE, P.MTX_REDUCE_ZERO1):
            gpu = run_model(rank, world, cfg, X, y, 2, P.MTX_FP32, mode)
            net = oracle.Net.from_cfg(cfg)
            w0 = oracle.init_params(net, 42)
            v0 = np.zeros_like(w0)
            for t, (rec, g) in enumerate(zip(recs, gpu)):
                check(abs(g[0] - rec.loss) <= 1e-5 * abs(rec.loss), f"mode {mode} step {t} loss")
                e = step_errors(net, cfg, X, y, t, w0, v0, g, world)
                check(max(e.values()) <= 1e-5, f"mode {mode} step {t} errors {e}")
                w0, v0 = g[2], g[3]
            check(maxrel(gpu[-1][2], w_ref) <= 1e-5, f"mode {mode} weights")
        report["checks"].append(f"layerwise and zero1 steps vs oracle at P={world}")

        # ---- FUSED (NVLink peer-memory reduce + update) is bit-exact with ORDERED (same rank-ordered fold)
        for prec in ([P.MTX_FP32, P.MTX_3XTF32, P.MTX_3XF16] if "tcgen05" in mtx.mtx_build_info() else [P.MTX_FP32]):
            # 3xF16 + cfg4's shape: the fused update's per-rank maxima give the same parameter planes as ORDERED's
            # own max pass
            for name, B, n in (("cfg1", 64, 1000), ("cfg2", 512, 4096)) + ((("cfg4", 512, 2048),) if prec == P.MTX_3XF16 else ()):
                cfg = dict(S.CONFIGS[name], B=B)
                X, y = S.higgs_like(1, n) if name == "cfg4" else S.mnist_like(1, n)
                a = run_model(rank, world, cfg, X, y, 3, prec, P.MTX_REDUCE_ORDERED)
                b = run_model(rank, world, cfg, X, y, 3, prec, P.MTX_REDUCE_FUSED)
                for t, ((la, Ga, wa, va), (lb, Gb, wb, vb)) in enumerate(zip(a, b)):
                    check(np.array_equal(Ga.view(np.uint32), Gb.view(np.uint32)), f"FUSED != ORDERED G {name} step {t}")
                    check(np.array_equal(wa.view(np.uint32), wb.view(np.uint32)), f"FUSED != ORDERED w {name} step {t}")
                    check(np.array_equal(va.view(np.uint32), vb.view(np.uint32)), f"FUSED != ORDERED v {name} step {t}")
                    check(la == lb, f"FUSED != ORDERED loss {name} step {t}: {la} {lb}")
        report["checks"].append(f"fused == ordered bitwise at P={world}")
        # ---- ORDERED reduce reproduces NCCL at P = 2
        if world == 2:
            cfg = dict(S.CONFIGS["cfg1"], B=64)
            X, y = S.mnist_like(1, 1000)
            a = run_model(rank, world, cfg, X, y, 2, P.MTX_FP32, P.MTX_REDUCE_NCCL)
            b = run_model(rank, world, cfg, X, y, 2, P.MTX_FP32, P.MTX_REDUCE_ORDERED)
            for (la, Ga, wa, _), (lb, Gb, wb, _) in zip(a, b):
                check(np.array_equal(Ga.view(np.uint32), Gb.view(np.uint32)), "ORDERED != NCCL G at P=2")
                check(np.array_equal(wa.view(np.uint32), wb.view(np.uint32)), "ORDERED != NCCL w at P=2")
            report["checks"].append("ordered == nccl at P=2")
        report["ok"] = True
    except Exception:  # noqa: BLE001
        report["ok"] = False
        report["error"] = traceback.format_exc()
    reports = allgather_obj(report)
    if rank == 0:
        path = os.environ.get("MTX_MP_REPORT")
        if path:
            json.dump(reports, open(path, "w"), indent=1)
        print(json.dumps(reports, indent=1))
    dist.destroy_process_group()
    sys.exit(0 if all(r["ok"] for r in reports) else 1)


if __name__ == "__main__":
    main()
