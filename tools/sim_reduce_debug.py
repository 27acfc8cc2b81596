"""Development probe: mtx_debug_reduce on simulated ranks -- where does it differ from the oracle?"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import mtx_synth as S  # noqa: E402
import oracle  # noqa: E402
import paper_1704_04560_b200 as P  # noqa: E402

r = P.Replica(dict(S.CONFIGS["cfg1"], B=4))
for mode in (P.MTX_REDUCE_ORDERED, P.MTX_REDUCE_FUSED):
    for Pn in (1, 2, 4):
        n = 4096
        g = np.zeros((Pn, n + 32), np.float32)
        for q in range(Pn):
            g[q, :n] = S.cfg5_grad_random(1, q, n)
        w, v = S.cfg5_params(1, n), S.cfg5_velocity(1, n)
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        gd, wd, vd = [dev(g[q]) for q in range(Pn)], [dev(w) for _ in range(Pn)], [dev(v) for _ in range(Pn)]
        Gd = [torch.zeros(n + 32, device="cuda") for _ in range(Pn)]
        torch.cuda.synchronize()
        t0 = time.time()
        P.mtx.mtx_debug_reduce(r.ctx, mode, Pn, [t.data_ptr() for t in gd], [t.data_ptr() for t in wd],
                               [t.data_ptr() for t in vd], [t.data_ptr() for t in Gd], n, 0.01, 0.9, r.s)
        r.sync()
        dt = time.time() - t0
        G = oracle.fold(g)
        wo, vo = w.copy(), v.copy()
        oracle.avg_update(G[:n].copy(), wo, vo, Pn, 0.01, 0.9)
        fl = torch.zeros(1, dtype=torch.int32)
        try:
            r.get()
            flag = "ok"
        except P.MtxError as e:
            flag = str(e)
        for q in range(Pn):
            wq = wd[q].cpu().numpy()
            bad = np.nonzero(wq.view(np.uint32) != wo.view(np.uint32))[0]
            same_as_w0 = np.nonzero(wq.view(np.uint32) == w.view(np.uint32))[0]
            Gq = Gd[q].cpu().numpy()
            gbad = np.nonzero(Gq[:n].view(np.uint32) != G[:n].view(np.uint32))[0]
            print(f"mode {mode} P {Pn} rank {q}: {dt*1e3:.1f} ms flag={flag} w bad {len(bad)} "
                  f"[{bad[:3]}..{bad[-3:] if len(bad) else ''}] unchanged {len(same_as_w0)}; G bad {len(gbad)} "
                  f"[{gbad[:3]}..]", flush=True)
r.close()
