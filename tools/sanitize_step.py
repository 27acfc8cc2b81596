"""Small product-path workload for compute-sanitizer (one tool per run): a cfg1 MLP step
and a LeNet step on the 3xTF32 tensor-core engines, the FP32 SIMT step, and the P = 2 fused NVLink protocol
on simulated ranks.  Prints one line per part."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mtx_synth as S  # noqa: E402
import paper_1704_04560_b200 as P  # noqa: E402

for prec in (P.MTX_3XTF32, P.MTX_FP32):
    for name, cfg, data in (("cfg1", dict(S.CONFIGS["cfg1"], B=64), S.mnist_like(1, 256)),
                            ("cfg3", dict(S.CONFIGS["cfg3"], B=16, n=64), S.cifar_like(1, 64))):
        r = P.Replica(cfg, precision=prec)
        r.bcast()
        r.shard(*data)
        for _ in range(2):
            loss = r.step(want_loss=True)
        r.close()
        print(f"{name} prec={prec} loss={loss:.6f}", flush=True)
r = P.Replica(dict(S.CONFIGS["cfg1"], B=4))
n, Pn = 4096, 2
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
g = [dev(np.concatenate([S.cfg5_grad_random(1, q, n), np.zeros(32, np.float32)])) for q in range(Pn)]
w = [dev(S.cfg5_params(1, n)) for _ in range(Pn)]
v = [dev(S.cfg5_velocity(1, n)) for _ in range(Pn)]
G = [torch.zeros(n + 32, device="cuda") for _ in range(Pn)]
torch.cuda.synchronize()
P.mtx.mtx_debug_reduce(r.ctx, P.MTX_REDUCE_FUSED, Pn, [t.data_ptr() for t in g], [t.data_ptr() for t in w],
                       [t.data_ptr() for t in v], [t.data_ptr() for t in G], n, 0.01, 0.9, r.s)
r.sync()
r.get()
r.close()
print("fused P=2 simulated ok", flush=True)
