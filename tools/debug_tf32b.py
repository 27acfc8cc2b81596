import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mtx_synth as S, oracle
import paper_1704_04560_b200 as P
from paper_1704_04560_b200 import mtx
from tests._util import per_tensor_maxrel, maxrel
rep = P.Replica(dict(S.CONFIGS["cfg4"], B=1024), precision=1)
rng = np.random.default_rng(0)
for (M, N, K, ta, tb) in [(64, 128, 784, 0, 0), (64, 128, 96, 0, 0), (100, 128, 64, 0, 0), (784, 128, 64, 1, 0), (784, 128, 32, 1, 0), (64, 784, 128, 0, 1)]:
    A = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    B = rng.standard_normal((N, K) if tb else (K, N)).astype(np.float32)
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    Ad, Bd = d(A), d(B); Cd = torch.full((M, N), np.nan, device="cuda"); torch.cuda.synchronize()
    mtx.mtx_debug_gemm(rep.ctx, 1, M, N, K, ta, tb, 0, Ad.data_ptr(), M if ta else K, Bd.data_ptr(), K if tb else N, Cd.data_ptr(), N, None, None, 0, rep.s)
    rep.sync()
    ref = (A.T if ta else A).astype(np.float64) @ (B.T if tb else B).astype(np.float64)
    C = Cd.cpu().numpy()
    print((M, N, K, ta, tb), "err %.2e" % maxrel(C, ref), "nan", np.isnan(C).sum(), "rows bad", np.where(np.abs(C - ref).max(1) > 1e-2 * np.abs(ref).max())[0][:10])
rep.close()
