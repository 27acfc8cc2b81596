import torch, time
n = 512*784*4
for sz in [n, 4*n, 16*n]:
    h = torch.empty(sz, dtype=torch.uint8).pin_memory(); d = torch.empty(sz, dtype=torch.uint8, device="cuda")
    for _ in range(5): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(100): d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1)/100
    # two streams, halves
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(100):
        with torch.cuda.stream(s1): d[:sz//2].copy_(h[:sz//2], non_blocking=True)
        with torch.cuda.stream(s2): d[sz//2:].copy_(h[sz//2:], non_blocking=True)
    torch.cuda.synchronize(); t2 = (time.perf_counter()-t0)*1e3/100
    print(f"{sz/1e6:.1f} MB: 1 stream {t*1e3:.1f} us = {sz/t/1e6:.1f} GB/s; 2 streams {t2*1e3:.1f} us = {sz/t2/1e6:.1f} GB/s")
