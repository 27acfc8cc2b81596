import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mtx_synth as S, oracle
import paper_1704_04560_b200 as P
from paper_1704_04560_b200 import mtx
from tests._util import per_tensor_maxrel
cfg = dict(S.CONFIGS["cfg1"], B=64)
X, y = S.mnist_like(1, 1000)
net = oracle.Net.from_cfg(cfg); tab = oracle.tensor_table(net)
start = oracle.init_params(net, 42)
for step in (0, 15):
    g_ref, l_ref = oracle.local_grad(net, start.astype(np.float64), X, y, 64, step, 0, 1)
    for prec in (0, 1):
        for bb in (0, 1 << 20):
            r = P.Replica(cfg, precision=prec, bucket_bytes=bb)
            r.bcast(); r.set(P.MTX_BUF_PARAMS, start); r.shard(X, y); r.step_idx = step
            loss = r.step(want_loss=True)
            G = r.get(P.MTX_BUF_GRADS); r.close()
            print("step", step, "prec", prec, "bucket", bb, "loss %.6f ref %.6f" % (loss, l_ref / 64), ["%.1e" % e for e in per_tensor_maxrel(G, g_ref, tab)])
