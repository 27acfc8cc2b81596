"""B200-native synchronous data-parallel SGD step of MaTEx-TensorFlow (arXiv 1704.04560).

The product is ``libmtx.so`` (C-ABI in ``include/mtx.h``); ``mtx`` is its thin
ctypes binding.  ``Replica`` below only marshals: it asks the library how much
device memory it needs, allocates that with PyTorch, lends it, and forwards the
calls.  One Replica per process per GPU (``torchrun``), NCCL for the data path,
a gloo process group only to ship the 128-byte NCCL unique id.
"""
from __future__ import annotations

import numpy as np

from . import mtx
from .mtx import (MTX_3XF16, MTX_3XTF32, MTX_BUF_GRADS, MTX_DEBUG_REDUCE_PUSH, MTX_BUF_PARAMS, MTX_BUF_VELOCITY, MTX_FP32,  # noqa: F401
                  MTX_REDUCE_FUSED, MTX_REDUCE_LAYERWISE, MTX_REDUCE_NCCL, MTX_REDUCE_ORDERED, MTX_REDUCE_ZERO1,
                  MTX_TF32, MtxError)

__all__ = ["mtx", "Replica", "MtxError", "nccl_uid_broadcast"]


def nccl_uid_broadcast(rank: int, world: int) -> bytes | None:
    """Rank 0 creates the NCCL unique id; it reaches the other ranks over torch.distributed (gloo)."""
    if world == 1:
        return None
    import torch
    import torch.distributed as dist
    uid = mtx.mtx_get_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    dist.broadcast(t, src=0)
    return bytes(t.tolist())


class Replica:
    """One rank's replica: context + torch-owned workspace + device-resident dataset."""

    def __init__(self, cfg: dict, rank: int = 0, world: int = 1, uid: bytes | None = None, device: int = 0,
                 precision: int = MTX_FP32, reduce: int = MTX_REDUCE_NCCL, bucket_bytes: int = 0,
                 init_seed: int = 42, B: int | None = None, lr: float | None = None, momentum: float | None = None):
        import torch
        self.torch = torch
        self.cfg = cfg
        self.rank, self.world, self.device = rank, world, device
        self.B = B if B is not None else cfg["B"]
        self.b = self.B // world
        torch.cuda.set_device(device)
        self.stream = torch.cuda.Stream(device=device)
        self.model = mtx.model_desc(cfg, self.B)
        self.opt = mtx.optim_desc(cfg["lr"] if lr is None else lr, cfg["mu"] if momentum is None else momentum,
                                  precision, reduce, bucket_bytes, init_seed)
        self.ctx = mtx.mtx_init(rank, world, uid, device, self.model, self.opt)
        nb = mtx.mtx_workspace_bytes(self.ctx)
        self.ws = torch.empty(nb, dtype=torch.uint8, device=f"cuda:{device}")
        torch.cuda.synchronize(device)
        mtx.mtx_bind_workspace(self.ctx, self.ws.data_ptr(), nb)
        self.N = mtx.mtx_param_count(self.ctx)
        self.data = None
        self.step_idx = 0

    @property
    def s(self) -> int:
        return self.stream.cuda_stream

    def bcast(self, root: int = 0):
        mtx.mtx_bcast_params(self.ctx, root, self.s)
        self.stream.synchronize()

    def shard(self, X: np.ndarray, y: np.ndarray):
        """Registers the dataset (host numpy arrays); every rank passes the same full dataset."""
        X = np.ascontiguousarray(X, np.float32).reshape(X.shape[0], -1)
        y = np.ascontiguousarray(y, np.int32)
        n = X.shape[0]
        nb = mtx.mtx_dataset_bytes(self.ctx, n)
        self.data = self.torch.empty(nb, dtype=self.torch.uint8, device=f"cuda:{self.device}")
        self.torch.cuda.synchronize(self.device)
        mtx.mtx_shard_data(self.ctx, X.ctypes.data, y.ctypes.data, n, X.shape[1], 0, self.data.data_ptr(), nb,
                           self.s)
        self.n = n
        self.step_idx = 0

    def step(self, want_loss: bool = False):
        loss = mtx.mtx_train_step(self.ctx, self.step_idx, want_loss, self.s)
        self.step_idx += 1
        return loss

    def step_host(self, X_rows: np.ndarray, y_rows: np.ndarray) -> float:
        return mtx.mtx_train_step_host(self.ctx, X_rows.ctypes.data, y_rows.ctypes.data, self.s)

    def step_host_async(self, X_rows: np.ndarray, y_rows: np.ndarray) -> None:
        """Pipelined host-input step (rows must stay valid and unchanged until sync_host())."""
        mtx.mtx_train_step_host_async(self.ctx, X_rows.ctypes.data, y_rows.ctypes.data, self.s)

    def sync_host(self) -> float:
        """Waits for the pipelined steps; returns the last step's global loss."""
        return mtx.mtx_sync(self.ctx, self.s)

    def sync(self):
        self.stream.synchronize()

    def get(self, which: int = MTX_BUF_PARAMS) -> np.ndarray:
        self.sync()
        return mtx.mtx_get_buffer(self.ctx, which)

    def set(self, which: int, values: np.ndarray):
        self.sync()
        mtx.mtx_set_buffer(self.ctx, which, values)

    def digest(self) -> int:
        self.sync()
        return mtx.mtx_param_digest(self.ctx)

    def close(self):
        if getattr(self, "ctx", None) is not None:
            self.sync()
            mtx.mtx_finalize(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
