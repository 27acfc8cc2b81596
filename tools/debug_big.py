import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import mtx_synth as S
import paper_1704_04560_b200 as P
from paper_1704_04560_b200 import mtx
rep = P.Replica(dict(S.CONFIGS["cfg4"]), precision=P.MTX_3XTF32)
for (M, N, K, ta, tb, epi) in [(8192, 1024, 1024, 0, 0, 1), (8192, 1024, 1024, 0, 1, 3), (1024, 1024, 8192, 1, 0, 0),
                               (28, 1024, 8192, 1, 0, 0), (8192, 1024, 28, 0, 0, 1), (1024, 1024, 1024, 0, 0, 1), (2048, 1024, 1024, 0, 0, 1), (4096, 1024, 1024, 0, 0, 1)]:
    A = torch.randn((K, M) if ta else (M, K), device="cuda")
    B = torch.randn((N, K) if tb else (K, N), device="cuda")
    bias = torch.randn(N, device="cuda"); mask = torch.randn(M, N, device="cuda")
    a = (A.t() if ta else A).double(); b = (B.t() if tb else B).double()
    ref = a @ b
    if epi == 1: ref = torch.relu(ref + bias.double())
    if epi == 3: ref = torch.where(mask > 0, ref, torch.zeros_like(ref))
    out = []
    for engine in (0, 1, 2):
        C = torch.full((M, N), float("nan"), device="cuda"); torch.cuda.synchronize()
        mtx.mtx_debug_gemm(rep.ctx, engine, M, N, K, ta, tb, epi, A.data_ptr(), M if ta else K, B.data_ptr(), K if tb else N, C.data_ptr(), N, bias.data_ptr(), mask.data_ptr(), N, rep.s)
        rep.sync()
        err = ((C.double() - ref).abs().max() / ref.abs().max()).item()
        bad = ((C.double() - ref).abs() > 1e-2 * ref.abs().max())
        rows = torch.nonzero(bad.any(1)).flatten()
        out.append("e%d %.1e nan%d badrows%d first%s" % (engine, err, int(torch.isnan(C).sum()), len(rows), rows[:3].tolist()))
    print((M, N, K, ta, tb, epi), out, flush=True)
rep.close()
