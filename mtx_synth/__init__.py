"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no forward/backward, no
reduction, no update, no parameter init). It only produces the *inputs* the
paper's workloads consume, shaped like them, from a counter-based generator, so
that the oracle (`oracle/`) and the CUDA path (`paper_1704_04560_b200/`) can be
fed bit-identical bytes without either importing the other.

Recipe:

* ``H(key, k)`` is the k-th output (0-based) of SplitMix64 seeded with ``key``
  (Steele, Lea, Flood, "Fast splittable pseudorandom number generators",
  OOPSLA 2014; Vigna's public-domain ``splitmix64.c``):
  ``z = key + (k+1)*0x9E3779B97F4A7C15; z = (z^(z>>30))*0xBF58476D1CE4E5B9;
  z = (z^(z>>27))*0x94D049BB133111EB; return z^(z>>31)`` (all mod 2^64).
* Stream keys ``K(seed, tag) = H(seed, tag)``: tag 1 labels, 2 values,
  3 class templates, 4+64r cfg5 gradients of rank r, 5 cfg5 velocity.
* MNIST-shaped (d=784, C=10), CIFAR-shaped (NHWC 32x32x3, C=10) and
  HIGGS-shaped (d=28, C=2) rows; every value is an integer mapped to fp32 by one
  correctly-rounded IEEE operation, so bytes are platform independent.

The paper's workloads are MNIST/CIFAR/ImageNet-style image classifiers and HEP
tabular data; the real files are not
available (no network), so these generators reproduce their shapes, label
balance and value ranges only.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

TAG_LABELS = 1
TAG_VALUES = 2
TAG_TEMPLATES = 3
TAG_CFG5_GRAD = 4
TAG_CFG5_VEL = 5


def splitmix64(key, k):
    """Vectorised H(key, k): k-th SplitMix64 output of a generator seeded with key."""
    with np.errstate(over="ignore"):
        key = np.uint64(key)
        k = np.asarray(k, dtype=np.uint64)
        z = key + (k + np.uint64(1)) * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def stream_key(seed: int, tag: int) -> np.uint64:
    return np.uint64(splitmix64(np.uint64(seed), np.uint64(tag)))


# --------------------------------------------------------------------------- datasets
MNIST_D, MNIST_C = 784, 10
CIFAR_H, CIFAR_W, CIFAR_CH, CIFAR_C = 32, 32, 3, 10
HIGGS_D, HIGGS_C = 28, 2

_CHUNK_ROWS = 1 << 16


def mnist_like(seed: int, n: int):
    """[n,784] fp32 in [0,1] + int32 labels in [0,10); ~19% non-zero strokes per class template."""
    ky, kv, kt = (stream_key(seed, t) for t in (TAG_LABELS, TAG_VALUES, TAG_TEMPLATES))
    y = (splitmix64(ky, np.arange(n, dtype=np.uint64)) % np.uint64(10)).astype(np.int32)
    tmpl = (splitmix64(kt, np.arange(10 * 784, dtype=np.uint64)) % np.uint64(5) == 0).reshape(10, 784)
    X = np.empty((n, 784), dtype=np.float32)
    for r0 in range(0, n, _CHUNK_ROWS):
        r1 = min(n, r0 + _CHUNK_ROWS)
        idx = (np.arange(r0, r1, dtype=np.uint64)[:, None] * np.uint64(784)
               + np.arange(784, dtype=np.uint64)[None, :])
        u = splitmix64(kv, idx)
        on = np.uint64(255) - (u % np.uint64(96))
        noise = np.where(((u >> np.uint64(8)) % np.uint64(100)) < np.uint64(3),
                         (u >> np.uint64(16)) % np.uint64(256), np.uint64(0))
        p = np.where(tmpl[y[r0:r1]], on, noise).astype(np.float32)
        X[r0:r1] = p / np.float32(255.0)
    return X, y


def cifar_like(seed: int, n: int):
    """[n,32,32,3] NHWC fp32 in [0,1] + int32 labels; per-class base colour + uniform jitter."""
    ky, kv, kt = (stream_key(seed, t) for t in (TAG_LABELS, TAG_VALUES, TAG_TEMPLATES))
    y = (splitmix64(ky, np.arange(n, dtype=np.uint64)) % np.uint64(10)).astype(np.int32)
    base = (np.uint64(64) + splitmix64(kt, np.arange(30, dtype=np.uint64)) % np.uint64(128)).astype(np.int64).reshape(10, 3)
    d = 32 * 32 * 3
    X = np.empty((n, 32, 32, 3), dtype=np.float32)
    ch = np.arange(d) % 3
    for r0 in range(0, n, _CHUNK_ROWS // 4):
        r1 = min(n, r0 + _CHUNK_ROWS // 4)
        idx = (np.arange(r0, r1, dtype=np.uint64)[:, None] * np.uint64(d)
               + np.arange(d, dtype=np.uint64)[None, :])
        u = splitmix64(kv, idx)
        p = base[y[r0:r1]][:, ch] + (u % np.uint64(97)).astype(np.int64) - 48
        p = np.clip(p, 0, 255).astype(np.float32)
        X[r0:r1] = (p / np.float32(255.0)).reshape(r1 - r0, 32, 32, 3)
    return X, y


def higgs_like(seed: int, n: int):
    """[n,28] fp32 ~N(0,1.15) (Irwin-Hall of four 16-bit uniforms) with class-shifted means; ~53% signal."""
    ky, kv = stream_key(seed, TAG_LABELS), stream_key(seed, TAG_VALUES)
    y = ((splitmix64(ky, np.arange(n, dtype=np.uint64)) % np.uint64(100)) < np.uint64(53)).astype(np.int32)
    shift = ((np.arange(28) % 7) - 3).astype(np.float32) / np.float32(16.0)
    X = np.empty((n, 28), dtype=np.float32)
    m = np.uint64(0xFFFF)
    for r0 in range(0, n, _CHUNK_ROWS * 4):
        r1 = min(n, r0 + _CHUNK_ROWS * 4)
        idx = (np.arange(r0, r1, dtype=np.uint64)[:, None] * np.uint64(28)
               + np.arange(28, dtype=np.uint64)[None, :])
        u = splitmix64(kv, idx)
        v = ((u & m) + ((u >> np.uint64(16)) & m) + ((u >> np.uint64(32)) & m) + (u >> np.uint64(48))).astype(np.int64)
        x = (v - 131070).astype(np.float32) / np.float32(32768.0)
        X[r0:r1] = x + np.where(y[r0:r1, None] == 1, shift[None, :], np.float32(0.0))
    return X, y


DATASETS = {"mnist": mnist_like, "cifar": cifar_like, "higgs": higgs_like}


# --------------------------------------------------------------------------- cfg5 buffers
def cfg5_grad_dyadic(seed: int, rank: int, n: int) -> np.ndarray:
    """Dyadic fp32 gradients ((u mod 2^21) - 2^20) * 2^-8: any summation order of <=8 ranks is exact."""
    k = stream_key(seed, TAG_CFG5_GRAD + 64 * rank)
    u = splitmix64(k, np.arange(n, dtype=np.uint64))
    return ((u % np.uint64(1 << 21)).astype(np.int64) - (1 << 20)).astype(np.float32) * np.float32(2.0 ** -8)


def cfg5_grad_random(seed: int, rank: int, n: int) -> np.ndarray:
    """Random-magnitude fp32 gradients sign * 2^e * (1 + m/2^23), e in [-20, 0]."""
    k = stream_key(seed, TAG_CFG5_GRAD + 64 * rank)
    u = splitmix64(k, np.arange(n, dtype=np.uint64))
    mant = (u & np.uint64((1 << 23) - 1)).astype(np.float64)
    e = ((u >> np.uint64(23)) % np.uint64(21)).astype(np.int64) - 20
    sgn = np.where((u >> np.uint64(63)) == 1, -1.0, 1.0)
    return (sgn * np.ldexp(1.0 + mant / 2.0 ** 23, e)).astype(np.float32)


def cfg5_velocity(seed: int, n: int) -> np.ndarray:
    """Dyadic fp32 velocity ((u mod 2^21) - 2^20) * 2^-27, |v| < 2^-7."""
    k = stream_key(seed, TAG_CFG5_VEL)
    u = splitmix64(k, np.arange(n, dtype=np.uint64))
    return ((u % np.uint64(1 << 21)).astype(np.int64) - (1 << 20)).astype(np.float32) * np.float32(2.0 ** -27)


def cfg5_params(seed: int, n: int) -> np.ndarray:
    """Parameter values for the flat-buffer sweep: uniform in [-0.05, 0.05) on a 2^-24 grid (input only)."""
    k = stream_key(seed, 6)
    u = splitmix64(k, np.arange(n, dtype=np.uint64)) >> np.uint64(40)
    return ((u.astype(np.float64) * 2.0 ** -24 * 2.0 - 1.0) * 0.05).astype(np.float32)


# --------------------------------------------------------------------------- configs
CONFIGS = {
    # BASELINE.json configs[0..4]; hyper-parameters per SURVEY.md §8(c) A20.
    "cfg1": dict(kind="mlp", dims=[784, 128, 10], data="mnist", n=1000, B=64, P=2, steps=5, lr=0.1, mu=0.0),
    "cfg2": dict(kind="mlp", dims=[784, 512, 512, 10], data="mnist", n=60000, B=512, steps=200, lr=0.01, mu=0.9),
    "cfg3": dict(kind="cnn", in_hwc=(32, 32, 3), conv=[(5, 6), (5, 16)], fc=[120, 84, 10], data="cifar",
                 n=50000, B=1024, steps=100, lr=0.01, mu=0.9),
    "cfg4": dict(kind="mlp", dims=[28, 1024, 1024, 1024, 1024, 2], data="higgs", n=10_000_000, B=8192,
                 steps=100, lr=0.01, mu=0.9),
}
DATA_SEED = 1
INIT_SEED = 42


def dataset(cfg: dict, n: int | None = None, seed: int = DATA_SEED):
    return DATASETS[cfg["data"]](seed, cfg["n"] if n is None else n)
