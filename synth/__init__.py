"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the oracle tests, the product tests and bench.py. It
holds none of the method's arithmetic: it only builds integer inverse-CDF
tables for three byte distributions and asks synth.c to turn counter-based
SplitMix64 draws into bytes.

Workloads (paper ``tab:datasets`` P:440-463):

* ``exp``   -- rand_lambda: byte = min(255, floor(256 X)), X ~ Exp(rate lambda)
               (reading Z22 of SURVEY.md; "random exponentially distributed bytes").
* ``text``  -- i.i.d. Zipf(s) over 96 printable ASCII bytes in a fixed English-like
               rank order; s = 1.0574 gives ~5.09 bit/byte (enwik8-like).
* ``image`` -- image-residual-like: zigzag(round(Laplace(0, b))) clipped to +-127,
               b log-uniform in [0.15, 3] quantised to 64 levels (marginal ~2.33 bit/byte,
               matching div2k801's 2,093/7,209 KB = 2.32 bit/byte at n=16), chosen per 64 KiB tile.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.c")
_LIB = os.path.join(_HERE, "libsynth.so")
_lib = None

TWO64 = 1 << 64


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-pthread",
                               _SRC, "-o", _LIB])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.synth_fill.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int]
        lib.synth_fill.restype = ctypes.c_int
        lib.synth_u64.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        lib.synth_u64.restype = None
        _lib = lib
    return _lib


def _thresholds(pmf) -> list[int]:
    """pmf over byte values 0..255 -> 256 non-decreasing 2^64-scaled cumulative thresholds."""
    total = float(sum(pmf))
    thr, acc = [], 0.0
    for k in range(256):
        acc += pmf[k] / total
        thr.append(min(TWO64 - 1, int(round(min(acc, 1.0) * TWO64))))
    thr[255] = TWO64 - 1
    for k in range(1, 256):  # enforce monotonicity against rounding
        thr[k] = max(thr[k], thr[k - 1])
    return thr


def exp_pmf(lam: float) -> list[float]:
    cdf = [1.0 - math.exp(-lam * (k + 1) / 256.0) for k in range(256)]
    cdf[255] = 1.0
    return [cdf[0]] + [cdf[k] - cdf[k - 1] for k in range(1, 256)]


TEXT_ORDER = (" etaoinshrdlcumwfgypbvkjxqz" + ",.\nETAOINSHRDLCUMWFGYPBVKJXQZ" +
              "0123456789" + "'\"-;:!?()[]/&*%$#@+=<>_|{}~^`\\\t")


def text_pmf(s: float = 1.0574) -> list[float]:
    chars = []
    for c in TEXT_ORDER:
        if ord(c) not in chars:
            chars.append(ord(c))
    chars = chars[:96]
    pmf = [0.0] * 256
    for r, c in enumerate(chars, start=1):
        pmf[c] = r ** (-s)
    return pmf


def laplace_residual_pmf(b: float) -> list[float]:
    """P(zigzag(clip(round(Laplace(0,b)), -127, 127)) = k)."""
    def cdf(x):  # Laplace(0, b) CDF
        return 0.5 * math.exp(x / b) if x < 0 else 1.0 - 0.5 * math.exp(-x / b)
    pmf = [0.0] * 256
    for v in range(-127, 128):
        lo = -math.inf if v == -127 else v - 0.5
        hi = math.inf if v == 127 else v + 0.5
        p = (1.0 if hi == math.inf else cdf(hi)) - (0.0 if lo == -math.inf else cdf(lo))
        z = 2 * v if v >= 0 else -2 * v - 1
        pmf[z] += p
    return pmf


IMAGE_LEVELS = 64
IMAGE_TILE = 1 << 16


def _tables_array(pmfs) -> np.ndarray:
    arr = np.zeros((len(pmfs), 256), dtype=np.uint64)
    for i, p in enumerate(pmfs):
        arr[i, :] = np.array(_thresholds(p), dtype=np.uint64)
    return arr


def _fill(n: int, seed: int, tables: np.ndarray, tile: int = 0, start: int = 0, threads: int | None = None):
    lib = _load()
    out = np.empty(int(n), dtype=np.uint8)
    if n == 0:
        return out
    tables = np.ascontiguousarray(tables, dtype=np.uint64)
    if threads is None:
        threads = max(1, min(16, os.cpu_count() or 1))
    lib.synth_fill(out.ctypes.data, start, int(n), seed & (TWO64 - 1), tables.ctypes.data,
                   tables.shape[0], tile, threads)
    return out


def exp_bytes(n: int, lam: float, seed: int) -> np.ndarray:
    return _fill(n, seed, _tables_array([exp_pmf(lam)]))


def text_bytes(n: int, seed: int, s: float = 1.0574) -> np.ndarray:
    return _fill(n, seed, _tables_array([text_pmf(s)]))


def image_bytes(n: int, seed: int) -> np.ndarray:
    levels = [0.15 * (20.0 ** (l / (IMAGE_LEVELS - 1))) for l in range(IMAGE_LEVELS)]
    return _fill(n, seed, _tables_array([laplace_residual_pmf(b) for b in levels]), tile=IMAGE_TILE)


def table_bytes(n: int, pmf, seed: int) -> np.ndarray:
    """Bytes i.i.d. from an arbitrary pmf over 0..255 (fuzz inputs)."""
    return _fill(n, seed, _tables_array([pmf]))


def u64(count: int, seed: int, start: int = 0) -> np.ndarray:
    lib = _load()
    out = np.empty(int(count), dtype=np.uint64)
    if count:
        lib.synth_u64(out.ctypes.data, start, int(count), seed & (TWO64 - 1))
    return out


def seed_for(config_id: int, lam: float = 0) -> int:
    """seed = 0x5EC011 + config_id*1000 + lambda."""
    return 0x5EC011 + config_id * 1000 + int(lam)


def workload(kind: str, n: int, seed: int, lam: float = 50.0) -> np.ndarray:
    if kind == "exp":
        return exp_bytes(n, lam, seed)
    if kind == "text":
        return text_bytes(n, seed)
    if kind == "image":
        return image_bytes(n, seed)
    raise ValueError(kind)


def histogram(sym: np.ndarray) -> np.ndarray:
    return np.bincount(sym, minlength=256).astype(np.uint64)
