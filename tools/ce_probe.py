"""Copy-engine (cudaMemcpyPeerAsync) NVLink probe, one process driving all visible GPUs.

Measures push bandwidth GPU0 -> peers for several sizes, the all-to-all push aggregate, and how much a tensor-core
GEMM on the source GPU slows down while its copy engines push.  Development measurement for the overlapped
reduction design; not a product path.
"""
import time
import torch

n = torch.cuda.device_count()
print("gpus", n)
devs = [torch.device("cuda", i) for i in range(n)]
MB = 1 << 20


def ev(d):
    return torch.cuda.Event(enable_timing=True)


def push_time(sizes, srcs, reps=20):
    out = {}
    for sz in sizes:
        nel = sz // 4
        bufs = {i: torch.empty(nel * n, device=devs[i]) for i in range(n)}
        streams = {(s, d): torch.cuda.Stream(device=devs[s]) for s in srcs for d in range(n) if d != s}
        for _ in range(3):
            for (s, d), st in streams.items():
                with torch.cuda.stream(st):
                    bufs[d][s * nel:(s + 1) * nel].copy_(bufs[s][d * nel:(d + 1) * nel], non_blocking=True)
        for i in range(n):
            torch.cuda.synchronize(devs[i])
        t0 = time.perf_counter()
        for _ in range(reps):
            for (s, d), st in streams.items():
                with torch.cuda.stream(st):
                    bufs[d][s * nel:(s + 1) * nel].copy_(bufs[s][d * nel:(d + 1) * nel], non_blocking=True)
        for i in range(n):
            torch.cuda.synchronize(devs[i])
        dt = (time.perf_counter() - t0) / reps
        per_src_out = sz * (n - 1) if len(srcs) else 0
        out[sz] = (dt * 1e6, per_src_out / dt / 1e9)
    return out


sizes = [256 * 1024, MB, 4 * MB, 16 * MB]
# single pair
for sz in sizes:
    nel = sz // 4
    a = torch.empty(nel, device=devs[0]); b = torch.empty(nel, device=devs[1])
    for _ in range(3): b.copy_(a, non_blocking=True)
    torch.cuda.synchronize(devs[0]); torch.cuda.synchronize(devs[1])
    e0, e1 = ev(0), ev(0)
    with torch.cuda.device(0):
        e0.record()
        for _ in range(20): b.copy_(a, non_blocking=True)
        e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    print(f"pair push 0->1 {sz/MB:7.2f} MB: {us:8.1f} us  {sz/us/1e3:7.1f} GB/s")
    a = torch.empty(nel, device=devs[1]); b = torch.empty(nel, device=devs[0])
    with torch.cuda.device(0):
        e0.record()
        for _ in range(20): b.copy_(a, non_blocking=True)
        e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    print(f"pair pull 1->0 {sz/MB:7.2f} MB: {us:8.1f} us  {sz/us/1e3:7.1f} GB/s")
r = push_time(sizes, [0])
for sz, (us, gbs) in r.items():
    print(f"GPU0 -> all peers concurrently {sz/MB:7.2f} MB each: {us:8.1f} us wall, {gbs:7.1f} GB/s out of GPU0")
r = push_time(sizes, list(range(n)))
for sz, (us, gbs) in r.items():
    print(f"all-to-all push {sz/MB:7.2f} MB per pair: {us:8.1f} us wall, {gbs:7.1f} GB/s out per GPU")

# GEMM slowdown under CE traffic (bf16 2048x1024x1024 chain on GPU0)
with torch.cuda.device(0):
    A = torch.randn(2048, 1024, device=devs[0], dtype=torch.bfloat16)
    W = torch.randn(1024, 1024, device=devs[0], dtype=torch.bfloat16)
    for _ in range(5): A @ W
    torch.cuda.synchronize()
    e0, e1 = ev(0), ev(0)
    e0.record()
    for _ in range(200): A @ W
    e1.record(); torch.cuda.synchronize()
    alone = e0.elapsed_time(e1) * 1e3 / 200
    nel = 4 * MB // 4
    srcb = torch.empty(nel * n, device=devs[0])
    dst = {d: torch.empty(nel, device=devs[d]) for d in range(1, n)}
    sts = {d: torch.cuda.Stream(device=devs[0]) for d in range(1, n)}
    e0.record()
    for _ in range(200): A @ W
    e1.record()
    for rep in range(40):
        for d, st in sts.items():
            with torch.cuda.stream(st):
                dst[d].copy_(srcb[d * nel:(d + 1) * nel], non_blocking=True)
    torch.cuda.synchronize()
    busy = e0.elapsed_time(e1) * 1e3 / 200
    print(f"bf16 GEMM 2048x1024x1024: alone {alone:.2f} us, with CE pushes to {n-1} peers {busy:.2f} us")
