"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws per-rank input buffers
(numpy PCG64, seed 20181113 + rank) in the shapes, sizes and
value distributions of the paper's workload (ResNet-50 gradients; FP16
communication).  The recipe is stated in DESIGN.md Sec. 4.

Storage conventions match ``oracle``: f32 -> float32, f16 -> float16, bf16 -> uint16 bit
patterns, i32 -> int32.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 20181113  # arXiv submission date of 1811.05233; SURVEY C12

# torchvision resnet50: 161 parameter tensors, 25,557,032 elements.
RESNET50_NUMEL = 25_557_032

STORAGE = {"f32": np.float32, "f16": np.float16, "bf16": np.uint16, "i32": np.int32}


def rng(rank: int, salt: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + rank + 1000 * salt))


def _f32_to_storage(x: np.ndarray, dtype: str) -> np.ndarray:
    """Store float32 draws in the buffer type.  f16 uses numpy's RNE cast; bf16 uses
    torch's RNE cast (CPU) -- input generation, not the method's arithmetic."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if dtype == "f32":
        return x
    if dtype == "f16":
        return x.astype(np.float16)
    if dtype == "bf16":
        import torch
        return torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16).copy()
    raise ValueError(dtype)


def make(dist: str, D: int, rank: int, dtype: str, salt: int = 0) -> np.ndarray:
    """One rank's input buffer of D elements.

    dist:
      uniform : U[0,1)                       (non-negative: |ref| == sum|x|)
      normal  : N(0,1)
      wide    : sign * N(0,1) * 10^U(-4,4)   (exercises association order)
      grad    : N(0,1) * 2^-7 -- ResNet-50-like gradient magnitudes (includes f16 subnormals)
      full    : i32 uniform over the whole int32 range (exercises wrap-around)
      onehot  : i32 1 << rank  (routing pin: sum is 2^N - 1 iff each rank counted once)
      ramp    : i32 rank * D + i  (closed-form pin)
      rank    : value == rank  (SPEC.md:231 worked example)
    """
    g = rng(rank, salt)
    if dtype == "i32":
        if dist == "full":
            return g.integers(-(2 ** 31), 2 ** 31, size=D, dtype=np.int64).astype(np.int32)
        if dist == "onehot":
            return np.full(D, 1 << rank, dtype=np.int32)
        if dist == "ramp":
            return (np.int64(rank) * D + np.arange(D, dtype=np.int64)).astype(np.int32)
        if dist == "rank":
            return np.full(D, rank, dtype=np.int32)
        if dist == "small":
            return g.integers(-1000, 1000, size=D, dtype=np.int64).astype(np.int32)
        raise ValueError(f"unknown i32 distribution {dist}")
    if dist == "uniform":
        x = g.random(D, dtype=np.float32)
    elif dist == "normal":
        x = g.standard_normal(D, dtype=np.float32)
    elif dist == "wide":
        sign = np.where(g.random(D) < 0.5, -1.0, 1.0)
        x = (sign * np.abs(g.standard_normal(D)) * 10.0 ** g.uniform(-4, 4, D)).astype(np.float32)
    elif dist == "grad":
        x = (g.standard_normal(D, dtype=np.float32) * np.float32(2.0 ** -7)).astype(np.float32)
    elif dist == "rank":
        x = np.full(D, rank, dtype=np.float32)
    else:
        raise ValueError(f"unknown float distribution {dist}")
    return _f32_to_storage(x, dtype)


def make_all(dist: str, D: int, N: int, dtype: str, salt: int = 0) -> list[np.ndarray]:
    return [make(dist, D, r, dtype, salt) for r in range(N)]


def as_float64(a: np.ndarray, dtype: str) -> np.ndarray:
    """Decode a storage array to float64 for error metrics (bf16: bit shift)."""
    if dtype == "bf16":
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


def resnet50_param_numels() -> list[int]:
    """torchvision resnet50 parameter sizes in registration order (161 tensors,
    25,557,032 elements), computed from the architecture without building the model."""
    sizes: list[int] = []

    def conv(cin, cout, k):
        sizes.append(cout * cin * k * k)

    def bn(c):
        sizes.extend([c, c])

    conv(3, 64, 7); bn(64)
    cin = 64
    for width, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        for b in range(blocks):
            cout = width * 4
            conv(cin, width, 1); bn(width)
            conv(width, width, 3); bn(width)
            conv(width, cout, 1); bn(cout)
            if b == 0:
                conv(cin, cout, 1); bn(cout)
            cin = cout
    sizes.extend([1000 * 2048, 1000])
    return sizes
