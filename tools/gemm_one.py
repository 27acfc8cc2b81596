"""One tcgen05 GEMM shape, repeated (for ncu): python tools/gemm_one.py M N K ta tb epi engine [reps]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mtx_synth as S
import paper_1704_04560_b200 as P
from paper_1704_04560_b200 import mtx
M, N, K, ta, tb, epi, engine = map(int, sys.argv[1:8])
reps = int(sys.argv[8]) if len(sys.argv) > 8 else 5
rep = P.Replica(dict(S.CONFIGS["cfg4"], B=1024), precision=P.MTX_3XTF32)
A = torch.randn((K, M) if ta else (M, K), device="cuda"); B = torch.randn((N, K) if tb else (K, N), device="cuda")
C = torch.empty(M, N, device="cuda"); bias = torch.randn(N, device="cuda"); mask = torch.randn(M, N, device="cuda")
for _ in range(reps):
    mtx.mtx_debug_gemm(rep.ctx, engine, M, N, K, ta, tb, epi, A.data_ptr(), M if ta else K, B.data_ptr(), K if tb else N,
                       C.data_ptr(), N, bias.data_ptr(), mask.data_ptr(), N, rep.s)
rep.sync(); rep.close(); print("ok")
