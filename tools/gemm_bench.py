"""Times the tcgen05 TF32 engine (mtx_debug_gemm) against cuBLAS TF32 (torch.matmul, context only)
on the step's shapes.  Prints one JSON line per shape."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mtx_synth as S
import paper_1704_04560_b200 as P
from paper_1704_04560_b200 import mtx

rep = P.Replica(dict(S.CONFIGS["cfg4"], B=1024), precision=P.MTX_3XTF32)
shapes = [(8192, 1024, 1024, 0, 0, 1), (8192, 1024, 1024, 0, 1, 3), (1024, 1024, 8192, 1, 0, 0),
          (8192, 1024, 28, 0, 0, 1), (512, 512, 784, 0, 0, 1), (784, 512, 512, 1, 0, 0), (4096, 4096, 4096, 0, 0, 1)]
torch.backends.cuda.matmul.allow_tf32 = True
for (M, N, K, ta, tb, epi) in shapes:
    A = torch.randn((K, M) if ta else (M, K), device="cuda")
    B = torch.randn((N, K) if tb else (K, N), device="cuda")
    C = torch.empty(M, N, device="cuda")
    bias = torch.randn(N, device="cuda")
    mask = torch.randn(M, N, device="cuda")
    s = rep.stream
    def run(engine):
        mtx.mtx_debug_gemm(rep.ctx, engine, M, N, K, ta, tb, epi, A.data_ptr(), M if ta else K, B.data_ptr(),
                           K if tb else N, C.data_ptr(), N, bias.data_ptr(), mask.data_ptr(), N, rep.s)
    res = {"M": M, "N": N, "K": K, "ta": ta, "tb": tb, "epi": epi}
    for engine in (1, 2, 0):
        if engine == 0 and M * N * K > 2e10:
            continue
        for _ in range(3):
            run(engine)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(20):
                run(engine)
            e1.record(s)
        s.synchronize()
        t = e0.elapsed_time(e1) / 20
        res[f"engine{engine}_us"] = round(t * 1e3, 2)
        res[f"engine{engine}_tflops"] = round(2 * M * N * K / t / 1e9, 1)
    a = A.t() if ta else A
    b = B.t() if tb else B
    for _ in range(3):
        torch.matmul(a, b)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20
    res["cublas_tf32_us"] = round(t * 1e3, 2)
    res["cublas_tf32_tflops"] = round(2 * M * N * K / t / 1e9, 1)
    print(json.dumps(res), flush=True)
rep.close()
