"""Seeded synthetic inputs shared by the tests, the oracle legs and bench.py.

This module holds NONE of the method's arithmetic (no offset composition, no set
algebra, no stencil or product): only input generators, so that the oracle side
and the CUDA side can be fed identical bits.  Recipes:

* ``uniform(seed, shape, dtype)`` — counter-based splitmix64 stream, element c
  (row-major linear index) gets h = splitmix64(seed*GOLDEN + c); fp64 = (h>>11)*2^-53,
  fp32 = (h>>40)*2^-24 (both in [0,1)); bf16 = (k-128)/128 with k = h>>56
  (exactly representable, in [-1, 1)); ints = low bits.
* ``random_bits(seed, shape, dtype)`` — raw splitmix64 bits (NaNs, denormals and
  infinities included) for raw-copy parity.
* ``eigenmode2d / eigenmode3d`` — Dirichlet eigenmodes with a zero ghost ring.
* ``harmonic2d / harmonic3d`` — integer discrete-harmonic fields (fixed points).
* ``int_bf16(seed, shape, lo, hi)`` — integer matrices stored as bf16 bit patterns.
* ``special_values(seed, shape, dtype)`` — ``uniform`` in [-1, 1) with about one cell in
  eight replaced by +Inf, +-0, subnormals, tiny or huge normals (no -Inf, so no stencil
  sum is Inf - Inf = NaN, whose bit pattern differs between x86 and the GPU).
* Standard seed of config i: ``SEED0 + i`` (SEED0 = 180905657).
"""
from __future__ import annotations

import numpy as np

SEED0 = 180905657
GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_stream(seed: int, start: int, count: int) -> np.ndarray:
    """h[c] = splitmix64(seed*GOLDEN + c) for c in [start, start+count)."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed % (1 << 64)) * GOLDEN
        x = base + np.arange(start, start + count, dtype=np.uint64)
        z = x + GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _hash(seed, shape, chunk=1 << 24):
    n = int(np.prod(shape))
    out = np.empty(n, np.uint64)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        out[s:e] = splitmix64_stream(seed, s, e - s)
    return out.reshape(shape)


def uniform(seed: int, shape, dtype: str = "f64") -> np.ndarray:
    h = _hash(seed, shape)
    if dtype == "f64":
        return (h >> np.uint64(11)).astype(np.float64) * 2.0**-53
    if dtype == "f32":
        return ((h >> np.uint64(40)).astype(np.float64) * 2.0**-24).astype(np.float32)
    if dtype == "bf16":  # returns uint16 bit patterns of exact values (k-128)/128
        k = (h >> np.uint64(56)).astype(np.int64)
        f = ((k - 128).astype(np.float32) / np.float32(128.0)).astype(np.float32)
        return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    if dtype == "i32":
        return (h & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    if dtype == "i64":
        return h.view(np.int64)
    raise ValueError(dtype)


def random_bits(seed: int, shape, dtype: str) -> np.ndarray:
    h = _hash(seed, shape)
    if dtype in ("f64", "i64"):
        return h.view(np.float64 if dtype == "f64" else np.int64)
    if dtype in ("f32", "i32"):
        return (h & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32 if dtype == "f32" else np.int32)
    if dtype == "bf16":
        return (h & np.uint64(0xFFFF)).astype(np.uint16)
    raise ValueError(dtype)


def int_bf16(seed: int, shape, lo: int = -4, hi: int = 4) -> np.ndarray:
    """integers uniformly in [lo, hi] as bf16 bit patterns (exact for |v| <= 256)."""
    h = _hash(seed, shape)
    v = (h % np.uint64(hi - lo + 1)).astype(np.int64) + lo
    f = v.astype(np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def eigenmode2d(n0: int, n1: int, a: int, b: int) -> np.ndarray:
    """u[i,j] = sin(a*pi*i/(n0-1)) * sin(b*pi*j/(n1-1)); ghost ring exactly 0."""
    i = np.arange(n0, dtype=np.float64)[:, None]
    j = np.arange(n1, dtype=np.float64)[None, :]
    u = np.sin(a * np.pi * i / (n0 - 1)) * np.sin(b * np.pi * j / (n1 - 1))
    u[0, :] = u[-1, :] = 0.0
    u[:, 0] = u[:, -1] = 0.0
    return np.ascontiguousarray(u)


def eigenmode3d(n0: int, n1: int, n2: int, a: int, b: int, c: int, dtype=np.float32) -> np.ndarray:
    z = np.arange(n0, dtype=np.float64)[:, None, None]
    y = np.arange(n1, dtype=np.float64)[None, :, None]
    x = np.arange(n2, dtype=np.float64)[None, None, :]
    u = (np.sin(a * np.pi * z / (n0 - 1)) * np.sin(b * np.pi * y / (n1 - 1))
         * np.sin(c * np.pi * x / (n2 - 1)))
    u[0], u[-1] = 0.0, 0.0
    u[:, 0], u[:, -1] = 0.0, 0.0
    u[:, :, 0], u[:, :, -1] = 0.0, 0.0
    return np.ascontiguousarray(u.astype(dtype))


def harmonic2d(n0: int, n1: int, dtype=np.float64) -> np.ndarray:
    """u = i^2 - j^2 (integer valued)."""
    i = np.arange(n0, dtype=np.int64)[:, None]
    j = np.arange(n1, dtype=np.int64)[None, :]
    return np.ascontiguousarray((i * i - j * j).astype(dtype))


def harmonic3d(n0: int, n1: int, n2: int, dtype=np.float32) -> np.ndarray:
    """u = z^2 + y^2 - 2 x^2 (integer valued)."""
    z = np.arange(n0, dtype=np.int64)[:, None, None]
    y = np.arange(n1, dtype=np.int64)[None, :, None]
    x = np.arange(n2, dtype=np.int64)[None, None, :]
    return np.ascontiguousarray((z * z + y * y - 2 * x * x).astype(dtype))


def special_values(seed: int, shape, dtype: str = "f64") -> np.ndarray:
    """uniform(seed) mapped to [-1, 1), with cells whose hash byte selects a special
    value: +Inf, +0, -0, the smallest subnormal, a mid subnormal, a tiny normal, a huge
    normal (positive and negative).  Edge cases of constant-weight divisions."""
    npdt = np.float64 if dtype == "f64" else np.float32
    u = uniform(seed, shape, dtype).astype(npdt) * npdt(2) - npdt(1)
    sel = (_hash(seed + 7, shape) >> np.uint64(56)).astype(np.int64)
    fi = np.finfo(npdt)
    specials = [np.inf, 0.0, -0.0, fi.smallest_subnormal, fi.smallest_normal * npdt(0.3),
                fi.smallest_normal * npdt(4), fi.max / npdt(64), -fi.max / npdt(64),
                fi.smallest_normal * npdt(2**30), -fi.smallest_normal * npdt(2**20)]
    for k, v in enumerate(specials):
        u[sel == 200 + 5 * k] = npdt(v)
        u[sel == 201 + 5 * k] = npdt(v)
        u[sel == 202 + 5 * k] = npdt(v)
    return u
