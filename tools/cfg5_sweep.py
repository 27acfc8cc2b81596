"""Config 5: the averaging operator on a flat fp32 gradient buffer, swept over sizes
(1 KB .. 256 MB, plus the AlexNet-scale 61,100,840-element point).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 tools/cfg5_sweep.py
    python tools/cfg5_sweep.py            # N = 1: the fused update (K6) alone

Per size, device-timed with CUDA events on the library's stream, max over ranks:
  * allreduce-only  (mtx_allreduce_avg apply_update = 0): algbw = 4n / t, busbw = algbw * 2(P-1)/P
  * allreduce + fused average/momentum update (apply_update = 1)
  * K6 alone on a world-1 context: achieved HBM GB/s = 20 n / t (momentum: G, w, v read; w, v write)
Buffers larger than L2 (126 MB) are streamed from HBM; smaller ones are marked "L2-resident".
Prints one JSON line per size (rank 0) and writes gpurun_out/cfg5_P<N>.jsonl.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import mtx_synth as S  # noqa: E402
import paper_1704_04560_b200 as P  # noqa: E402
from paper_1704_04560_b200 import mtx  # noqa: E402

SIZES = [256, 1 << 10, 1 << 12, 1 << 14, 1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24, 61_100_840, 1 << 26]


def timed(fn, s, iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(iters):
            fn()
        e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) / iters / 1e3


def main():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(local)
    tiny = dict(S.CONFIGS["cfg1"], B=4 * world)
    uid = P.nccl_uid_broadcast(rank, world)
    rep = P.Replica(tiny, rank=rank, world=world, uid=uid, device=local)
    solo = P.Replica(tiny, device=local)  # world-1 context: K6 alone
    out = []
    lr, mu = 0.01, 0.9
    for n in SIZES:
        G = torch.from_numpy(S.cfg5_grad_dyadic(1, rank, n)).cuda()
        w = torch.from_numpy(S.cfg5_params(1, n)).cuda()
        v = torch.from_numpy(S.cfg5_velocity(1, n)).cuda()
        torch.cuda.synchronize()
        iters = max(3, min(200, int(2e9 / (20 * n + 1e6))))
        res = {"n": n, "bytes": 4 * n, "P": world, "iters": iters, "l2_resident": 20 * n < 126e6}
        if world > 1:
            ar = lambda: mtx.mtx_allreduce_avg(rep.ctx, G.data_ptr(), None, None, n, lr, mu, 0, rep.s)
            full = lambda: mtx.mtx_allreduce_avg(rep.ctx, G.data_ptr(), w.data_ptr(), v.data_ptr(), n, lr, mu, 1,
                                                 rep.s)
            for f in (ar, full):
                for _ in range(3):
                    f()
            dist.barrier()
            t_ar = timed(ar, rep.stream, iters)
            dist.barrier()
            t_full = timed(full, rep.stream, iters)
            tt = torch.tensor([t_ar, t_full], dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_ar, t_full = float(tt[0]), float(tt[1])
            algbw = 4 * n / t_ar / 1e9
            res.update(allreduce_us=round(t_ar * 1e6, 2), algbw_gbs=round(algbw, 1),
                       busbw_gbs=round(algbw * 2 * (world - 1) / world, 1), allreduce_update_us=round(t_full * 1e6, 2))
        k6 = lambda: mtx.mtx_allreduce_avg(solo.ctx, G.data_ptr(), w.data_ptr(), v.data_ptr(), n, lr, mu, 1, solo.s)
        for _ in range(3):
            k6()
        t_k6 = timed(k6, solo.stream, iters)
        res.update(k6_us=round(t_k6 * 1e6, 3), k6_gbs=round(20 * n / t_k6 / 1e9, 1))
        # the values blow up after many momentum steps on the same G: reset (not timed)
        if rank == 0:
            print(json.dumps(res), flush=True)
        out.append(res)
        del G, w, v
        torch.cuda.empty_cache()
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"cfg5_P{world}.jsonl"), "w") as f:
            for r in out:
                f.write(json.dumps(r) + "\n")
    rep.close()
    solo.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
