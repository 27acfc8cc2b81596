"""Thin ctypes binding of include/mtx.h -- argument marshalling only.

Every function below has the C name and forwards to libmtx.so; every step of
the data-parallel SGD path runs in the library's sm_100a kernels and NCCL.
PyTorch is used only to allocate the device memory the library borrows and to
hand over streams.  There is no CPU fallback: if libmtx.so is missing or was
not built for this GPU, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmtx.so")

STATUS = ["MTX_OK", "MTX_ERR_INVALID_ARG", "MTX_ERR_STATE", "MTX_ERR_SHAPE", "MTX_ERR_CUDA", "MTX_ERR_NCCL",
          "MTX_ERR_NUMERIC", "MTX_ERR_PROTOCOL", "MTX_ERR_OOM", "MTX_ERR_UNSUPPORTED"]
MTX_MLP, MTX_CNN = 0, 1
MTX_FP32, MTX_TF32, MTX_3XTF32, MTX_3XF16 = 0, 1, 2, 3
MTX_REDUCE_NCCL, MTX_REDUCE_ORDERED, MTX_REDUCE_FUSED, MTX_REDUCE_LAYERWISE, MTX_REDUCE_ZERO1 = 0, 1, 2, 3, 4
MTX_BUF_PARAMS, MTX_BUF_VELOCITY, MTX_BUF_GRADS = 0, 1, 2
MTX_DEBUG_REDUCE_PUSH = 0x100  # mtx_debug_reduce: FUSED with the push protocol


class MtxError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str = ""):
        self.status = status
        name = STATUS[status] if 0 <= status < len(STATUS) else str(status)
        super().__init__(f"{where}: {name} {msg}".strip())


class mtx_model_desc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_dims", C.c_int32), ("dims", C.POINTER(C.c_int32)),
                ("in_h", C.c_int32), ("in_w", C.c_int32), ("in_c", C.c_int32),
                ("n_conv", C.c_int32), ("conv_k", C.POINTER(C.c_int32)), ("conv_c", C.POINTER(C.c_int32)),
                ("n_fc", C.c_int32), ("fc_dims", C.POINTER(C.c_int32)), ("global_batch", C.c_int64)]


class mtx_optim_desc(C.Structure):
    _fields_ = [("lr", C.c_float), ("momentum", C.c_float), ("precision", C.c_int32), ("reduce", C.c_int32),
                ("bucket_bytes", C.c_uint64), ("init_seed", C.c_uint64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(LIB_PATH)
    vp, u8p, f, i32, i64, u64 = C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_float), C.POINTER(C.c_int32), \
        C.POINTER(C.c_int64), C.POINTER(C.c_uint64)
    sigs = {
        "mtx_get_unique_id": [u8p],
        "mtx_init": [C.POINTER(vp), C.c_int32, C.c_int32, u8p, C.c_int32, C.POINTER(mtx_model_desc),
                     C.POINTER(mtx_optim_desc)],
        "mtx_workspace_bytes": [vp, u64],
        "mtx_bind_workspace": [vp, vp, C.c_uint64],
        "mtx_param_count": [vp, u64],
        "mtx_bcast_params": [vp, C.c_int32, vp],
        "mtx_dataset_bytes": [vp, C.c_int64, u64],
        "mtx_shard_data": [vp, vp, vp, C.c_int64, C.c_int64, C.c_int32, vp, C.c_uint64, vp],
        "mtx_batch_slice": [C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, i64, i64],
        "mtx_train_step": [vp, C.c_int64, f, vp],
        "mtx_train_step_host": [vp, vp, vp, f, vp],
        "mtx_train_step_host_async": [vp, vp, vp, vp],
        "mtx_sync": [vp, f, vp],
        "mtx_allreduce_avg": [vp, vp, vp, vp, C.c_uint64, C.c_float, C.c_float, C.c_int32, vp],
        "mtx_get_buffer": [vp, C.c_int32, f, C.c_uint64],
        "mtx_set_buffer": [vp, C.c_int32, f, C.c_uint64],
        "mtx_get_params": [vp, f, C.c_uint64],
        "mtx_get_loss": [vp, f],
        "mtx_param_digest": [vp, u64],
        "mtx_launches_per_step": [vp, i32],
        "mtx_set_timing": [vp, C.c_int32],
        "mtx_read_timing": [vp, C.c_char_p, C.c_uint64, C.POINTER(C.c_double), i64, C.c_int32, i32, C.c_int32],
        "mtx_finalize": [vp],
        "mtx_sync_update": [vp, vp],
        "mtx_debug_reduce": [vp, C.c_int32, C.c_int32, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), C.POINTER(vp),
                             C.c_uint64, C.c_float, C.c_float, vp],
        "mtx_debug_gemm": [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, vp,
                           C.c_int64, vp, C.c_int64, vp, C.c_int64, vp, vp, C.c_int64, vp],
    }
    for name, args in sigs.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    lib.mtx_last_error.argtypes = [vp]
    lib.mtx_last_error.restype = C.c_char_p
    lib.mtx_build_info.argtypes = []
    lib.mtx_build_info.restype = C.c_char_p
    return lib


_lib = _load()
EXPORTED = [n for n in dir(_lib) if n.startswith("mtx_")]


def _check(st: int, ctx, where: str):
    if st != 0:
        msg = _lib.mtx_last_error(ctx).decode() if ctx else ""
        raise MtxError(st, where, msg)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


# ------------------------------------------------------------------ same-name wrappers
def mtx_build_info() -> str:
    return _lib.mtx_build_info().decode()


def mtx_get_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    _check(_lib.mtx_get_unique_id(buf), None, "mtx_get_unique_id")
    return bytes(buf)


def mtx_init(rank: int, world: int, uid: bytes | None, device: int, model: mtx_model_desc, opt: mtx_optim_desc):
    ctx = C.c_void_p()
    ub = (C.c_uint8 * 128).from_buffer_copy(uid) if uid is not None else None
    st = _lib.mtx_init(C.byref(ctx), rank, world, ub, device, C.byref(model), C.byref(opt))
    _check(st, ctx if ctx.value else None, "mtx_init")
    return ctx


def mtx_workspace_bytes(ctx) -> int:
    v = C.c_uint64()
    _check(_lib.mtx_workspace_bytes(ctx, C.byref(v)), ctx, "mtx_workspace_bytes")
    return v.value


def mtx_bind_workspace(ctx, dev_ptr: int, nbytes: int):
    _check(_lib.mtx_bind_workspace(ctx, C.c_void_p(dev_ptr), nbytes), ctx, "mtx_bind_workspace")


def mtx_param_count(ctx) -> int:
    v = C.c_uint64()
    _check(_lib.mtx_param_count(ctx, C.byref(v)), ctx, "mtx_param_count")
    return v.value


def mtx_bcast_params(ctx, root: int = 0, stream: int | None = None):
    _check(_lib.mtx_bcast_params(ctx, root, C.c_void_p(stream)), ctx, "mtx_bcast_params")


def mtx_dataset_bytes(ctx, n: int) -> int:
    v = C.c_uint64()
    _check(_lib.mtx_dataset_bytes(ctx, n, C.byref(v)), ctx, "mtx_dataset_bytes")
    return v.value


def mtx_shard_data(ctx, X_ptr: int, y_ptr: int, n: int, sample_elems: int, src_is_device: int, dev_buf: int,
                   buf_bytes: int, stream: int | None = None):
    _check(_lib.mtx_shard_data(ctx, C.c_void_p(X_ptr), C.c_void_p(y_ptr), n, sample_elems, src_is_device,
                               C.c_void_p(dev_buf), buf_bytes, C.c_void_p(stream)), ctx, "mtx_shard_data")


def mtx_batch_slice(n: int, B: int, step: int, rank: int, world: int):
    b = (C.c_int64 * 2)()
    l = (C.c_int64 * 2)()
    _check(_lib.mtx_batch_slice(n, B, step, rank, world, b, l), None, "mtx_batch_slice")
    return (b[0], b[1]), (l[0], l[1])


def mtx_train_step(ctx, step: int, want_loss: bool = False, stream: int | None = None):
    loss = C.c_float()
    _check(_lib.mtx_train_step(ctx, step, C.byref(loss) if want_loss else None, C.c_void_p(stream)), ctx,
           "mtx_train_step")
    return loss.value if want_loss else None


def mtx_train_step_host(ctx, X_ptr: int, y_ptr: int, stream: int | None = None) -> float:
    loss = C.c_float()
    _check(_lib.mtx_train_step_host(ctx, C.c_void_p(X_ptr), C.c_void_p(y_ptr), C.byref(loss), C.c_void_p(stream)),
           ctx, "mtx_train_step_host")
    return loss.value


def mtx_train_step_host_async(ctx, X_ptr: int, y_ptr: int, stream: int | None = None) -> None:
    _check(_lib.mtx_train_step_host_async(ctx, C.c_void_p(X_ptr), C.c_void_p(y_ptr), C.c_void_p(stream)), ctx,
           "mtx_train_step_host_async")


def mtx_sync(ctx, stream: int | None = None) -> float:
    loss = C.c_float()
    _check(_lib.mtx_sync(ctx, C.byref(loss), C.c_void_p(stream)), ctx, "mtx_sync")
    return loss.value


def mtx_allreduce_avg(ctx, grad: int, param: int | None, velocity: int | None, count: int, lr: float,
                      momentum: float, apply_update: int = 1, stream: int | None = None):
    _check(_lib.mtx_allreduce_avg(ctx, C.c_void_p(grad), C.c_void_p(param), C.c_void_p(velocity), count, lr,
                                  momentum, apply_update, C.c_void_p(stream)), ctx, "mtx_allreduce_avg")


def mtx_sync_update(ctx, stream: int | None = None):
    _check(_lib.mtx_sync_update(ctx, C.c_void_p(stream)), ctx, "mtx_sync_update")


def mtx_get_buffer(ctx, which: int) -> np.ndarray:
    n = mtx_param_count(ctx)
    out = np.empty(n, np.float32)
    _check(_lib.mtx_get_buffer(ctx, which, _fp(out), n), ctx, "mtx_get_buffer")
    return out


def mtx_set_buffer(ctx, which: int, values: np.ndarray):
    v = np.ascontiguousarray(values, np.float32)
    _check(_lib.mtx_set_buffer(ctx, which, _fp(v), v.size), ctx, "mtx_set_buffer")


def mtx_get_params(ctx) -> np.ndarray:
    return mtx_get_buffer(ctx, MTX_BUF_PARAMS)


def mtx_get_loss(ctx) -> float:
    v = C.c_float()
    _check(_lib.mtx_get_loss(ctx, C.byref(v)), ctx, "mtx_get_loss")
    return v.value


def mtx_param_digest(ctx) -> int:
    v = C.c_uint64()
    _check(_lib.mtx_param_digest(ctx, C.byref(v)), ctx, "mtx_param_digest")
    return v.value


def mtx_launches_per_step(ctx) -> int:
    v = C.c_int32()
    _check(_lib.mtx_launches_per_step(ctx, C.byref(v)), ctx, "mtx_launches_per_step")
    return v.value


def mtx_set_timing(ctx, enable: bool):
    _check(_lib.mtx_set_timing(ctx, int(enable)), ctx, "mtx_set_timing")


def mtx_read_timing(ctx, reset: bool = True) -> dict:
    names = C.create_string_buffer(8192)
    ms = (C.c_double * 64)()
    cnt = (C.c_int64 * 64)()
    n = C.c_int32()
    _check(_lib.mtx_read_timing(ctx, names, 8192, ms, cnt, 64, C.byref(n), int(reset)), ctx, "mtx_read_timing")
    keys = names.value.decode().split("\n")[: n.value]
    return {k: (ms[i], cnt[i]) for i, k in enumerate(keys)}


def mtx_debug_gemm(ctx, engine, M, N, K, ta, tb, epi, A, lda, B, ldb, C, ldc, bias=None, mask=None, ldm=0,
                   stream=None):
    _check(_lib.mtx_debug_gemm(ctx, engine, M, N, K, ta, tb, epi, C_ptr(A), lda, C_ptr(B), ldb, C_ptr(C), ldc,
                               C_ptr(bias), C_ptr(mask), ldm, C_ptr(stream)), ctx, "mtx_debug_gemm")


def mtx_debug_reduce(ctx, mode, P, g, w, v, G, n, lr, momentum, stream=None):
    """g, w, v, G: sequences of P device addresses (v entries may be None when momentum == 0)."""
    arr = lambda xs: (C.c_void_p * P)(*[C.c_void_p(x) if x else None for x in xs])
    _check(_lib.mtx_debug_reduce(ctx, mode, P, arr(g), arr(w), arr(v if v is not None else [None] * P), arr(G), n,
                                 lr, momentum, C_ptr(stream)), ctx, "mtx_debug_reduce")


def C_ptr(x):
    return C.c_void_p(x)


def mtx_last_error(ctx) -> str:
    return _lib.mtx_last_error(ctx).decode()


def mtx_finalize(ctx):
    _check(_lib.mtx_finalize(ctx), None, "mtx_finalize")


# ------------------------------------------------------------------ descriptor helpers (marshalling)
def model_desc(cfg: dict, B: int | None = None) -> mtx_model_desc:
    """mtx_model_desc from a config dict (keys as in mtx_synth.CONFIGS)."""
    m = mtx_model_desc()
    keep = []

    def arr(x):
        a = (C.c_int32 * max(1, len(x)))(*x)
        keep.append(a)
        return C.cast(a, C.POINTER(C.c_int32))

    if cfg["kind"] == "mlp":
        m.kind, m.n_dims, m.dims = MTX_MLP, len(cfg["dims"]), arr(cfg["dims"])
        m.conv_k = m.conv_c = m.fc_dims = arr([0])
    else:
        h, w, c = cfg["in_hwc"]
        m.kind, m.in_h, m.in_w, m.in_c = MTX_CNN, h, w, c
        m.n_conv = len(cfg["conv"])
        m.conv_k, m.conv_c = arr([k for k, _ in cfg["conv"]]), arr([co for _, co in cfg["conv"]])
        m.n_fc, m.fc_dims = len(cfg["fc"]), arr(cfg["fc"])
        m.dims = arr([0])
    m.global_batch = B if B is not None else cfg["B"]
    m._keep = keep
    return m


def optim_desc(lr: float, momentum: float, precision: int = MTX_FP32, reduce: int = MTX_REDUCE_NCCL,
               bucket_bytes: int = 0, init_seed: int = 42) -> mtx_optim_desc:
    return mtx_optim_desc(lr, momentum, precision, reduce, bucket_bytes, init_seed)
