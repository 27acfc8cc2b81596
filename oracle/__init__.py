"""Oracle for the synchronous data-parallel SGD step -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_1704_04560_b200``) never imports it, and it never imports the product.

``mtx_oracle.c`` holds the arithmetic (plain C, IEEE double, -ffp-contract=off);
this file only marshals arguments and writes out the outer loop of the method
exactly as the paper states it:

  broadcast once, then per step:  shard (O4) -> local gradient on
  every simulated rank (O5-O7) -> ascending-rank left-fold allreduce-sum (O9,
  P:298-306) -> x fl(1/P) (O10) -> momentum update (O11), replicas kept as
  separate arrays so bit-identity (I2) is observable.

Inputs come from ``mtx_synth`` (seeded generators, no method arithmetic).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mtx_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC", "-shared"]


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (plain -O2, no contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


class _Net(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_dims", C.c_int32), ("dims", C.POINTER(C.c_int32)),
                ("in_h", C.c_int32), ("in_w", C.c_int32), ("in_c", C.c_int32),
                ("n_conv", C.c_int32), ("conv_k", C.POINTER(C.c_int32)), ("conv_c", C.POINTER(C.c_int32)),
                ("n_fc", C.c_int32), ("fc_dims", C.POINTER(C.c_int32))]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER
        d, f, i32, i64 = P(C.c_double), P(C.c_float), P(C.c_int32), P(C.c_int64)
        net = P(_Net)
        sig = {
            "orc_splitmix64": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "orc_param_count": (C.c_int64, [net]),
            "orc_tensor_table": (C.c_int, [net, i64, i64]),
            "orc_init_params": (None, [net, C.c_uint64, f]),
            "orc_batch_slice": (C.c_int, [C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, i64, i64]),
            "orc_local_grad": (C.c_double, [net, d, f, i32, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                            C.c_int32, d]),
            "orc_local_grad_tf32emu": (C.c_double, [net, d, f, i32, C.c_int64, C.c_int64, C.c_int64, C.c_int32,
                                                    C.c_int32, d]),
            "orc_mlp_activations_tf32emu": (None, [net, d, f, i32, C.c_int64, C.c_int, d]),
            "orc_tf32": (C.c_double, [C.c_double]),
            "orc_batch_grad": (C.c_double, [net, d, f, i32, C.c_int64, d]),
            "orc_mlp_activations": (None, [net, d, f, i32, C.c_int64, C.c_int, d]),
            "orc_fold_f64": (None, [C.c_int32, C.c_int64, d, d]),
            "orc_fold_f32": (None, [C.c_int32, C.c_int64, f, f]),
            "orc_avg_update_f64": (C.c_int64, [C.c_int64, C.c_int32, C.c_double, C.c_double, d, d, d]),
            "orc_avg_update_f32": (C.c_int64, [C.c_int64, C.c_int32, C.c_float, C.c_float, f, f, f]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype, fn.argtypes = res, args
    return _lib


def _ptr(a: np.ndarray, ct):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class Net:
    """MLP (``dims``) or LeNet-style CNN (``in_hwc``, ``conv`` [(k, c_out)], ``fc`` widths)."""
    kind: str = "mlp"
    dims: list = field(default_factory=list)
    in_hwc: tuple = (0, 0, 0)
    conv: list = field(default_factory=list)
    fc: list = field(default_factory=list)

    @staticmethod
    def from_cfg(cfg: dict) -> "Net":
        if cfg["kind"] == "mlp":
            return Net("mlp", list(cfg["dims"]))
        return Net("cnn", [], tuple(cfg["in_hwc"]), list(cfg["conv"]), list(cfg["fc"]))

    def c(self):
        # keep the arrays alive on the struct object
        arrs = [np.ascontiguousarray(x, dtype=np.int32) for x in
                (self.dims or [0], [k for k, _ in self.conv] or [0], [c for _, c in self.conv] or [0], self.fc or [0])]
        s = _Net(0 if self.kind == "mlp" else 1, len(self.dims), _ptr(arrs[0], C.c_int32),
                 self.in_hwc[0], self.in_hwc[1], self.in_hwc[2], len(self.conv), _ptr(arrs[1], C.c_int32),
                 _ptr(arrs[2], C.c_int32), len(self.fc), _ptr(arrs[3], C.c_int32))
        s._keep = arrs
        return s

    @property
    def classes(self) -> int:
        return self.dims[-1] if self.kind == "mlp" else self.fc[-1]

    @property
    def sample_elems(self) -> int:
        return self.dims[0] if self.kind == "mlp" else int(np.prod(self.in_hwc))


def splitmix64(key: int, k: int) -> int:
    return int(lib().orc_splitmix64(key, k))


def param_count(net: Net) -> int:
    return int(lib().orc_param_count(C.byref(net.c())))


def tensor_table(net: Net):
    off = np.zeros(64, np.int64)
    size = np.zeros(64, np.int64)
    n = lib().orc_tensor_table(C.byref(net.c()), _ptr(off, C.c_int64), _ptr(size, C.c_int64))
    return [(int(off[i]), int(size[i])) for i in range(n)]


def init_params(net: Net, seed: int) -> np.ndarray:
    """O2: fp32 Glorot-uniform init keyed by seed (rank r uses init_seed + r)."""
    out = np.zeros(param_count(net), np.float32)
    lib().orc_init_params(C.byref(net.c()), seed, _ptr(out, C.c_float))
    return out


def batch_slice(n: int, B: int, step: int, rank: int, P: int):
    """O4: (begin[2], len[2]) sample-id pieces of rank's shard at step."""
    b = np.zeros(2, np.int64)
    l = np.zeros(2, np.int64)
    rc = lib().orc_batch_slice(n, B, step, rank, P, _ptr(b, C.c_int64), _ptr(l, C.c_int64))
    if rc != 0:
        raise ValueError("invalid batch_slice arguments")
    return (int(b[0]), int(b[1])), (int(l[0]), int(l[1]))


def local_grad(net: Net, params: np.ndarray, X: np.ndarray, y: np.ndarray, B: int, step: int, rank: int, P: int,
               tf32emu: bool = False):
    """O5-O7 on rank's shard: (grad [N] f64 of the local MEAN loss, local loss SUM).
    tf32emu: the TF32 tier's contractions with A12-truncated operands (MLP only, readings A12/A23)."""
    params = np.ascontiguousarray(params, np.float64)
    X = np.ascontiguousarray(X, np.float32)
    y = np.ascontiguousarray(y, np.int32)
    g = np.zeros(param_count(net), np.float64)
    fn = lib().orc_local_grad_tf32emu if tf32emu else lib().orc_local_grad
    loss = fn(C.byref(net.c()), _ptr(params, C.c_double), _ptr(X, C.c_float), _ptr(y, C.c_int32), X.shape[0], B,
              step, rank, P, _ptr(g, C.c_double))
    return g, float(loss)


def tf32(x: float) -> float:
    """A12: an fp32 value as tcgen05 kind::tf32 consumes it (low 13 mantissa bits dropped)."""
    return float(lib().orc_tf32(float(x)))


def batch_grad(net: Net, params: np.ndarray, X: np.ndarray, y: np.ndarray, want_grad: bool = True):
    """Gradient of the mean loss over the explicit rows X (no sharding); returns (grad or None, loss sum)."""
    params = np.ascontiguousarray(params, np.float64)
    X = np.ascontiguousarray(X, np.float32)
    y = np.ascontiguousarray(y, np.int32)
    g = np.zeros(param_count(net), np.float64) if want_grad else None
    loss = lib().orc_batch_grad(C.byref(net.c()), _ptr(params, C.c_double), _ptr(X, C.c_float),
                                _ptr(y, C.c_int32), X.shape[0], _ptr(g, C.c_double) if want_grad else None)
    return g, float(loss)


def mlp_activations(net: Net, params, X, y, layer: int, tf32emu: bool = False) -> np.ndarray:
    params = np.ascontiguousarray(params, np.float64)
    X = np.ascontiguousarray(X, np.float32)
    y = np.ascontiguousarray(y, np.int32)
    out = np.zeros((X.shape[0], net.dims[layer]), np.float64)
    (lib().orc_mlp_activations_tf32emu if tf32emu else lib().orc_mlp_activations)(C.byref(net.c()), _ptr(params, C.c_double), _ptr(X, C.c_float), _ptr(y, C.c_int32),
                              X.shape[0], layer, _ptr(out, C.c_double))
    return out


def fold(gs: np.ndarray) -> np.ndarray:
    """O9: ascending-rank left fold of gs[P, N] (f64 or f32 by input dtype)."""
    gs = np.ascontiguousarray(gs)
    P, N = gs.shape
    if gs.dtype == np.float64:
        G = np.zeros(N, np.float64)
        lib().orc_fold_f64(P, N, _ptr(gs, C.c_double), _ptr(G, C.c_double))
    else:
        gs = gs.astype(np.float32)
        G = np.zeros(N, np.float32)
        lib().orc_fold_f32(P, N, _ptr(gs, C.c_float), _ptr(G, C.c_float))
    return G


def avg_update(G: np.ndarray, w: np.ndarray, v: np.ndarray, P: int, lr: float, mu: float) -> int:
    """O10-O11 in place on (w, v); fp32 (bit-exact definition) or f64 by dtype. Returns non-finite count."""
    N = G.shape[0]
    if G.dtype == np.float32:
        assert w.dtype == np.float32 and v.dtype == np.float32
        return int(lib().orc_avg_update_f32(N, P, np.float32(lr), np.float32(mu), _ptr(G, C.c_float),
                                            _ptr(w, C.c_float), _ptr(v, C.c_float)))
    return int(lib().orc_avg_update_f64(N, P, lr, mu, _ptr(G, C.c_double), _ptr(w, C.c_double),
                                        _ptr(v, C.c_double)))


@dataclass
class StepRecord:
    step: int
    loss: float           # global loss = (sum_r loss_sum_r) / B
    G: np.ndarray         # reduced (summed, not yet averaged) gradient
    grads: list           # per-rank local gradients g_r


def train(net: Net, X, y, B: int, P: int, steps: int, lr: float, mu: float, init_seed: int,
          keep_grads: bool = False, check_replicas: bool = True, start_params=None):
    """DP(P) simulation in f64 (SEQ is P=1).  Returns (records, params[f64], velocity[f64]).

    Broadcast (O3): every replica starts from rank 0's init (seed init_seed + 0), v = 0.
    """
    N = param_count(net)
    # O2: rank r initialises its own replica with seed init_seed + r ...
    if start_params is None:
        reps_w = [init_params(net, init_seed + r).astype(np.float64) for r in range(P)]
    else:
        reps_w = [np.array(start_params, np.float64) for _ in range(P)]
    # ... O3: then the Global Broadcast makes every replica rank 0's, bitwise.
    for r in range(1, P):
        reps_w[r][:] = reps_w[0]
    reps_v = [np.zeros(N, np.float64) for _ in range(P)]
    recs = []
    for t in range(steps):
        gs = np.zeros((P, N), np.float64)
        losses = np.zeros(P, np.float64)
        for r in range(P):
            gs[r], losses[r] = local_grad(net, reps_w[r], X, y, B, t, r, P)
        G = fold(gs)
        loss_sum = fold(losses.reshape(P, 1))[0]
        for r in range(P):  # every replica applies the same update to its own copy
            bad = avg_update(G, reps_w[r], reps_v[r], P, lr, mu)
            if bad:
                raise FloatingPointError(f"non-finite averaged gradient at step {t} ({bad} entries)")
        if check_replicas:
            for r in range(1, P):
                if reps_w[r].tobytes() != reps_w[0].tobytes() or reps_v[r].tobytes() != reps_v[0].tobytes():
                    raise AssertionError(f"replica {r} diverged from replica 0 at step {t}")
        recs.append(StepRecord(t, float(loss_sum / B), G if keep_grads else None, list(gs) if keep_grads else None))
    return recs, reps_w[0], reps_v[0]
