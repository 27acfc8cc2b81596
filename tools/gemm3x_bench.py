"""Times the tcgen05 3xTF32 engine on the step's GEMM shapes (mtx_debug_gemm engine 3: the contraction
alone, on precomputed hi/lo planes) against the 3xTF32 ceiling = measured bf16 burst x (1.1 / 2.25) / 3;
ENGINE=f16: the 3xF16 engine (engines 4/5) against its ceiling = measured bf16 burst / 3.
One JSON line per shape; LABEL names the plan knobs set in the environment (MTX_TC_PAIR_MASK, ...; the
library reads them once per process)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mtx_synth as S  # noqa: E402
import paper_1704_04560_b200 as P  # noqa: E402
from paper_1704_04560_b200 import mtx  # noqa: E402

pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
F16 = os.environ.get("ENGINE") == "f16"
ceil = pk["bf16_tflops"] / 3 if F16 else pk["bf16_tflops"] * 1.1 / 2.25 / 3
rep = P.Replica(dict(S.CONFIGS["cfg4"], B=1024), precision=P.MTX_3XF16 if F16 else P.MTX_3XTF32)
E0, E1 = (4, 5) if F16 else (2, 3)
shapes = [(8192, 1024, 1024, 0, 0, 1), (8192, 1024, 1024, 0, 1, 3), (1024, 1024, 8192, 1, 0, 0),
          (4096, 1024, 1024, 0, 0, 1), (4096, 1024, 1024, 0, 1, 3), (1024, 1024, 4096, 1, 0, 0),
          (2048, 1024, 1024, 0, 0, 1), (2048, 1024, 1024, 0, 1, 3), (1024, 1024, 2048, 1, 0, 0),
          (8192, 1024, 28, 0, 0, 1), (28, 1024, 8192, 1, 0, 0)]
only = os.environ.get("SHAPES")
for i, (M, N, K, ta, tb, epi) in enumerate(shapes):
    if only and str(i) not in only.split(","):
        continue
    A = torch.randn((K, M) if ta else (M, K), device="cuda")
    B = torch.randn((N, K) if tb else (K, N), device="cuda")
    C = torch.empty(M, N, device="cuda")
    bias = torch.randn(N, device="cuda")
    mask = torch.randn(M, N, device="cuda")
    s = rep.stream

    def run(engine):
        mtx.mtx_debug_gemm(rep.ctx, engine, M, N, K, ta, tb, epi, A.data_ptr(), M if ta else K, B.data_ptr(),
                           K if tb else N, C.data_ptr(), N, bias.data_ptr(), mask.data_ptr(), N, rep.s)
    for plan in [os.environ.get("LABEL", "default")]:
        run(E0)
        for _ in range(3):
            run(E1)
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(20):
                run(E1)
            e1.record(s)
        s.synchronize()
        t = e0.elapsed_time(e1) / 20
        ref = (A.t() if ta else A).double() @ (B.t() if tb else B).double()
        if epi == 1:
            ref = torch.relu(ref + bias.double())
        elif epi == 3:
            ref = torch.where(mask > 0, ref, torch.zeros_like(ref))
        err = ((C.double() - ref).abs().max() / ref.abs().max()).item()
        tf = 2 * M * N * K / t / 1e9
        print(json.dumps({"M": M, "N": N, "K": K, "ta": ta, "tb": tb, "epi": epi, "plan": plan, "us": round(t * 1e3, 2),
                          "tflops": round(tf, 1), "frac_3x_ceiling": round(tf / ceil, 3), "maxrel": err,
                          "engine": "3xf16" if F16 else "3xtf32", "dbg": os.environ.get("MTX_TC_DBG", "0")}), flush=True)
rep.close()
