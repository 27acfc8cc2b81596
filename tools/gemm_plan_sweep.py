"""Sweeps the tcgen05 GEMM tile plan (N tile x split-K) on the step's shapes: device time of one
contraction incl. its split-K fold, via mtx_debug_gemm engine 1 (TF32) / 3 (3xTF32, planes split
beforehand).  Prints one line per (shape, precision) with the time of every plan and the plan
tc_plan picks by default.  Development tool: drives MTX_TC_BN / MTX_TC_SPLITS."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mtx_synth as S
import paper_1704_04560_b200 as P
from paper_1704_04560_b200 import mtx

rep = P.Replica(dict(S.CONFIGS["cfg4"]), precision=P.MTX_3XTF32)  # full-size: split-K partial room
SHAPES = {  # (M, N, K, ta, tb, epi)
    "cfg2_fwd1": (512, 512, 784, 0, 0, 1), "cfg2_fwd2": (512, 512, 512, 0, 0, 1),
    "cfg2_dgrad": (512, 512, 512, 0, 1, 3), "cfg2_wgrad1": (784, 512, 512, 1, 0, 0),
    "cfg2_wgrad2": (512, 512, 512, 1, 0, 0),
    "cfg4_fwd": (8192, 1024, 1024, 0, 0, 1), "cfg4_dgrad": (8192, 1024, 1024, 0, 1, 3),
    "cfg4_wgrad": (1024, 1024, 8192, 1, 0, 0), "cfg4_fwd1": (8192, 1024, 28, 0, 0, 1),
    # fixed-cost probes: one tile / one k-block, and one tile with a deep K
    "tiny_1tile_1kb": (128, 64, 32, 0, 0, 0), "tiny_1tile_8kb": (128, 64, 256, 0, 0, 0),
    "tiny_148tiles_1kb": (128 * 37, 256, 32, 0, 0, 0),
}
only = sys.argv[1:] or list(SHAPES)


def timed(fn, iters=20):
    """Device time per call: `iters` calls captured in one CUDA graph (host launch cost excluded)."""
    for _ in range(2):
        fn(s.cuda_stream)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(iters):
            fn(cs.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * iters) * 1e3


s = torch.cuda.Stream()
for name in only:
    M, N, K, ta, tb, epi = SHAPES[name]
    A = torch.randn((K, M) if ta else (M, K), device="cuda")
    B = torch.randn((N, K) if tb else (K, N), device="cuda")
    C = torch.empty(M, N, device="cuda")
    bias = torch.randn(N, device="cuda")
    mask = torch.randn(M, N, device="cuda")
    lda, ldb = (M if ta else K), (K if tb else N)
    for eng, tag in ((1, "tf32"), (3, "3xtf32")):
        if eng == 3:  # split once (engine 2), then time engine 3
            mtx.mtx_debug_gemm(rep.ctx, 2, M, N, K, ta, tb, epi, A.data_ptr(), lda, B.data_ptr(), ldb,
                               C.data_ptr(), N, bias.data_ptr(), mask.data_ptr(), N, rep.s)
            torch.cuda.synchronize()
        run = lambda st: mtx.mtx_debug_gemm(rep.ctx, eng, M, N, K, ta, tb, epi, A.data_ptr(), lda, B.data_ptr(),
                                            ldb, C.data_ptr(), N, bias.data_ptr(), mask.data_ptr(), N, st)
        os.environ.pop("MTX_TC_BN", None); os.environ.pop("MTX_TC_SPLITS", None)
        res = {"shape": name, "prec": tag, "default_us": round(timed(run), 2)}
        kb = (K + 31) // 32
        for bn in ((128, 64, 32) if not name.startswith("tiny") else ()):
            for sp in (1, 2, 3, 4, 6, 8, 12, 16):
                if sp > kb:
                    continue
                os.environ["MTX_TC_BN"], os.environ["MTX_TC_SPLITS"] = str(bn), str(sp)
                try:
                    res[f"{bn}x{sp}"] = round(timed(run), 2)
                except Exception as e:  # partial buffer too small etc.
                    res[f"{bn}x{sp}"] = None
        os.environ.pop("MTX_TC_BN", None); os.environ.pop("MTX_TC_SPLITS", None)
        best = min((v, k) for k, v in res.items() if k not in ("shape", "prec") and v)
        res["best"] = best[1]
        print(json.dumps(res), flush=True)
rep.close()
