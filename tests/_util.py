"""Shared test helpers (comparison metrics; no method arithmetic)."""
from __future__ import annotations

import numpy as np

# Tolerance tier (BASELINE.json north_star; max-norm relative error per tensor, A21):
#   MTX_FP32 (0), MTX_3XTF32 (2) and MTX_3XF16 (3): 1e-5 -- the fp32 tier, gated on every gradient, loss
#   and weight.
# MTX_TF32 (1xTF32) is not a product precision (A22: its truncated operands leave
# 1e-2..2.4e-1 gradient errors, outside the north_star's 1e-3 TF32 tier) and has no entry here.
TOL = {0: 1e-5, 2: 1e-5, 3: 1e-5}
GRAD_TOL = {0: 1e-5, 2: 1e-5, 3: 1e-5}


def maxrel(x, ref) -> float:
    """Max-norm relative error: max_i |x_i - r_i| / max_i |r_i| (reading of "1e-5 relative")."""
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    den = max(np.abs(ref).max(initial=0.0), 1e-30)
    return float(np.abs(x - ref).max(initial=0.0) / den)


def per_tensor_maxrel(x, ref, table) -> list:
    return [maxrel(x[o:o + s], ref[o:o + s]) for o, s in table]


def digest_np(params: np.ndarray, vel: np.ndarray) -> int:
    """Recomputes mtx_param_digest's definition from host copies (include/mtx.h)."""
    import mtx_synth as S
    idx = np.arange(params.size, dtype=np.uint64)
    with np.errstate(over="ignore"):
        hp = S.splitmix64(0, 0)  # noqa: F841 (warm)
        a = _sm_keyvec(params.view(np.uint32).astype(np.uint64), idx)
        b = _sm_keyvec(vel.view(np.uint32).astype(np.uint64), idx + np.uint64(1 << 40))
        return int((a.sum(dtype=np.uint64) + b.sum(dtype=np.uint64)) & np.uint64(0xFFFFFFFFFFFFFFFF))


def _sm_keyvec(keys: np.ndarray, k: np.ndarray) -> np.ndarray:
    G = np.uint64(0x9E3779B97F4A7C15)
    z = keys + (k + np.uint64(1)) * G
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))
