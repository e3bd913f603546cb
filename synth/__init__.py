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
        lib.synth_fill_models.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_int]
        lib.synth_fill_models.restype = ctypes.c_int
        lib.synth_histogram.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int]
        lib.synth_histogram.restype = None
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


def exp_bytes(n: int, lam: float, seed: int, start: int = 0) -> np.ndarray:
    return _fill(n, seed, _tables_array([exp_pmf(lam)]), start=start)


def text_bytes(n: int, seed: int, s: float = 1.0574, start: int = 0) -> np.ndarray:
    return _fill(n, seed, _tables_array([text_pmf(s)]), start=start)


def image_bytes(n: int, seed: int, start: int = 0) -> np.ndarray:
    levels = [0.15 * (20.0 ** (l / (IMAGE_LEVELS - 1))) for l in range(IMAGE_LEVELS)]
    return _fill(n, seed, _tables_array([laplace_residual_pmf(b) for b in levels]), tile=IMAGE_TILE, start=start)


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


def workload(kind: str, n: int, seed: int, lam: float = 50.0, start: int = 0) -> np.ndarray:
    """Symbols [start, start + n) of the seeded stream (any sub-range is generated
    independently: the draws are counter-based)."""
    if kind == "exp":
        return exp_bytes(n, lam, seed, start)
    if kind == "text":
        return text_bytes(n, seed, start=start)
    if kind == "image":
        return image_bytes(n, seed, start)
    raise ValueError(kind)


def histogram(sym: np.ndarray) -> np.ndarray:
    """Byte histogram (256 x u64) of a uint8 array, multithreaded in synth.c."""
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    h = np.zeros(256, np.uint64)
    _load().synth_histogram(sym.ctypes.data, len(sym), h.ctypes.data, max(1, min(16, os.cpu_count() or 1)))
    return h


# --- latent workload: 16-bit symbols with index-keyed Gaussian models -------------------
# (div2k through mbt2018-mean, 16-bit symbols, each modelled by a Gaussian
# whose scale comes from the hyperprior; NEXT rows 1 + 4 of SURVEY.md §8(f)).
# The hyperprior itself is out of scope: scales are synthetic.  Recipe (DESIGN.md
# "Input recipe"): K = 64 scale classes sigma_k = exp(linspace(ln 0.11, ln 32, 64))
# (a compressai-style scale table, capped at 32); model k covers the residuals
# d in [-R_k, R_k], R_k = ceil(4.5 sigma_k) + 1, as 16-bit values 32768 + d; its
# integer histogram is the discretised Gaussian mass of each d (the two ends
# absorb the tails) scaled to 2^40, floored at 1.  Model ids: the flattened
# latent is C = 192 channels x 64 x 64; channel c has a base class a_c =
# floor(64 sqrt(u_c)), every 8 x 8 spatial tile t an
# offset b_t in {-4..4}; class = clamp(a_c + b_t, 0, 63).  Mean entropy ~4.4
# bit/symbol (div2k801 at n = 16: 2,093 KB of 7,209 KB = 4.64 bit/symbol, tab:datasets).

LATENT_K = 64
LATENT_CENTER = 32768
LATENT_C, LATENT_H, LATENT_W = 192, 64, 64


def latent_scales(K: int = LATENT_K) -> list[float]:
    return [math.exp(math.log(0.11) + (math.log(32.0) - math.log(0.11)) * k / (K - 1)) for k in range(K)]


def gaussian_hist(sigma: float) -> tuple[int, list[int]]:
    """-> (R, integer histogram over d = -R..R)."""
    R = int(math.ceil(4.5 * sigma)) + 1
    def Phi(x):
        return 0.5 * math.erfc(-x / math.sqrt(2.0))
    hist = []
    for d in range(-R, R + 1):
        lo = 0.0 if d == -R else Phi((d - 0.5) / sigma)
        hi = 1.0 if d == R else Phi((d + 0.5) / sigma)
        hist.append(max(1, int(round((hi - lo) * (1 << 40)))))
    return R, hist


def latent_model_hists(K: int = LATENT_K):
    """-> {"base": u32[K], "len": u32[K], "hist": [u64 array per model]}"""
    base, ln, hists = [], [], []
    for sg in latent_scales(K):
        R, h = gaussian_hist(sg)
        base.append(LATENT_CENTER - R)
        ln.append(2 * R + 1)
        hists.append(np.array(h, dtype=np.uint64))
    return {"base": np.array(base, dtype=np.uint32), "len": np.array(ln, dtype=np.uint32), "hist": hists}


def latent_model_ids(n: int, seed: int, K: int = LATENT_K) -> np.ndarray:
    """Per-index model ids (the decoder-side 'hyperprior' output), see the recipe above."""
    i = np.arange(int(n), dtype=np.int64)
    plane = LATENT_H * LATENT_W
    ch = i // plane                       # global channel counter (images repeat every C channels)
    y = (i % plane) // LATENT_W
    x = i % LATENT_W
    tile = ch * (plane // 64) + (y // 8) * (LATENT_W // 8) + (x // 8)
    n_ch = int(ch[-1]) + 1 if n else 0
    n_tile = int(tile.max()) + 1 if n else 0
    uc = u64(n_ch, seed ^ 0xA5A5A5A5) if n else np.zeros(0, np.uint64)
    ut = u64(n_tile, seed ^ 0x5A5A5A5A) if n else np.zeros(0, np.uint64)
    a = np.floor(K * np.sqrt((uc >> np.uint64(11)).astype(np.float64) / float(1 << 53))).astype(np.int64)
    b = (ut % np.uint64(9)).astype(np.int64) - 4
    return np.clip(a[ch] + b[tile], 0, K - 1).astype(np.uint8)


def latent_symbols(mid: np.ndarray, seed: int, hists=None, threads: int | None = None) -> np.ndarray:
    """16-bit symbols drawn from the models' integer histograms (exact inverse CDF)."""
    if hists is None:
        hists = latent_model_hists()
    thr, off = [], [0]
    for h in hists["hist"]:
        tot = int(h.sum())
        acc = 0
        for v in h.tolist():
            acc += int(v)
            thr.append(min(TWO64 - 1, (acc * TWO64) // tot))
        thr[-1] = TWO64 - 1
        off.append(off[-1] + len(h))
    thr = np.array(thr, dtype=np.uint64)
    off = np.array(off, dtype=np.uint64)
    base = np.ascontiguousarray(hists["base"], dtype=np.uint32)
    ln = np.ascontiguousarray(hists["len"], dtype=np.uint32)
    mid = np.ascontiguousarray(mid, dtype=np.uint8)
    out = np.empty(mid.size, dtype=np.uint16)
    if mid.size:
        if threads is None:
            threads = max(1, min(16, os.cpu_count() or 1))
        _load().synth_fill_models(out.ctypes.data, mid.ctypes.data, 0, mid.size, seed & (TWO64 - 1), thr.ctypes.data,
                                  off.ctypes.data, base.ctypes.data, ln.ctypes.data, threads)
    return out


def latent_workload(n: int, seed: int):
    """-> (symbols u16[n], model ids u8[n], model histograms)"""
    hists = latent_model_hists()
    mid = latent_model_ids(n, seed)
    return latent_symbols(mid, seed, hists), mid, hists
