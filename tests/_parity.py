"""One-step parity metric shared by the single- and multi-GPU tests (calls only oracle/)."""
from __future__ import annotations

import numpy as np

import oracle
from tests._util import per_tensor_maxrel


def step_errors(net, cfg, X, y, t, w0, v0, rec, P_=1):
    """One GPU step against the oracle started from the GPU's own state (w0, v0) before it, in f64:
    per-tensor max-norm relative error of the reduced gradient G, the loss, the velocity after the
    update (mu > 0: it carries the averaged gradient at full relative precision) and the weight
    change (less the single fp32 rounding of w_after, at most half an ulp)."""
    loss, G, w1, v1 = rec
    tab = oracle.tensor_table(net)
    gs, ls = zip(*[oracle.local_grad(net, w0.astype(np.float64), X, y, cfg["B"], t, r, P_) for r in range(P_)])
    G_ref = oracle.fold(np.stack(gs))
    lref = sum(ls) / cfg["B"]
    w_ref, v_ref = w0.astype(np.float64), v0.astype(np.float64)
    oracle.avg_update(G_ref, w_ref, v_ref, P_, cfg["lr"], cfg["mu"])
    dw, dw_ref = w1.astype(np.float64) - w0, w_ref - w0
    half_ulp = np.spacing(np.abs(w1)).astype(np.float64) / 2
    e_dw = [float(np.maximum(np.abs(dw[o:o + n] - dw_ref[o:o + n]) - half_ulp[o:o + n], 0).max(initial=0)
                  / max(np.abs(dw_ref[o:o + n]).max(initial=0), 1e-30)) for o, n in tab]
    return {"G": max(per_tensor_maxrel(G, G_ref, tab)), "loss": abs(loss - lref) / max(abs(lref), 1e-30),
            "v": max(per_tensor_maxrel(v1, v_ref, tab)) if cfg["mu"] else 0.0, "dw": max(e_dw)}
