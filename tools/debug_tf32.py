import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import mtx_synth as S, oracle
import paper_1704_04560_b200 as P
from paper_1704_04560_b200 import mtx
from tests._util import per_tensor_maxrel

cfg = dict(S.CONFIGS["cfg2"])
X, y = S.mnist_like(1, 4096)
net = oracle.Net.from_cfg(cfg); tab = oracle.tensor_table(net)
start = oracle.init_params(net, 42)
g_ref, _ = oracle.local_grad(net, start.astype(np.float64), X, y, 512, 0, 0, 1)
def run(prec, eager, **kw):
    r = P.Replica(cfg, precision=prec, **kw)
    r.bcast(); r.shard(X, y)
    if eager: mtx.mtx_set_timing(r.ctx, True)
    r.step(want_loss=True)
    G = r.get(P.MTX_BUF_GRADS); r.close(); return G
for prec in (0, 1):
    for eager in (False, True):
        G = run(prec, eager)
        print("prec", prec, "eager", eager, ["%.1e" % e for e in per_tensor_maxrel(G, g_ref, tab)])
# host-staged (no dataset offset) TF32
r = P.Replica(cfg, precision=1); r.bcast()
l = r.step_host(np.ascontiguousarray(X[:512]), np.ascontiguousarray(y[:512]))
G = r.get(P.MTX_BUF_GRADS); r.close()
print("tf32 staged", ["%.1e" % e for e in per_tensor_maxrel(G, g_ref, tab)])
