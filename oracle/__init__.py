"""TEST INFRASTRUCTURE ONLY -- ctypes wrapper of the plain C oracle (oracle.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with
``paper_2306_12141_b200`` (the product) and never imports it.

Parity status: every function here is pinned by
tests/test_oracle_pins.py except the container byte layout, which the paper
does not print ("parity unpinned": layout), and the quantiser
``build_model`` whose algorithm the paper does not give (pinned only
to its invariants and SPEC's worked examples).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
# ORACLE_SANITIZE=1: an ASan + UBSan build (tools/sanitize_host.sh) under its own name
_SAN = os.environ.get("ORACLE_SANITIZE") == "1"
_LIB = os.path.join(_HERE, "liboracle_san.so" if _SAN else "liboracle.so")
_lib = None

L = 1 << 16
ERRORS = {0: "OK", -1: "E_ARG", -2: "E_MODEL", -3: "E_UNDERFLOW", -4: "E_END", -5: "E_CONTAINER",
          -6: "E_NOMEM", -7: "E_BUFFER", -8: "E_OVERFLOW"}


class OracleError(RuntimeError):
    def __init__(self, rc):
        super().__init__(f"oracle error {rc} ({ERRORS.get(rc, '?')})")
        self.rc = rc


def build(force: bool = False) -> str:
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < newest:
        san = ["-fsanitize=address,undefined", "-fno-omit-frame-pointer", "-fno-sanitize-recover=undefined"] if _SAN \
            else []
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", *san, _SRC, "-o", _LIB])
    return _LIB


class Event(ctypes.Structure):
    _fields_ = [("idx", ctypes.c_int64), ("lane", ctypes.c_uint32), ("state", ctypes.c_uint32)]


EVENT_DTYPE = np.dtype([("idx", np.int64), ("lane", np.uint32), ("state", np.uint32)])

P = ctypes.c_void_p
U8P = ctypes.POINTER(ctypes.c_uint8)


def _load():
    global _lib
    if _lib is not None:
        return _lib
    build()
    lib = ctypes.CDLL(_LIB)
    u32, u64, i64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int
    sig = {
        "or_build_model": (i32, [P, u32, P]),
        "or_encode_step": (u64, [u64, u32, u32, u32]),
        "or_decode_step": (i32, [u32, P, u32, P, P]),
        "or_renorm_encode": (i32, [P, u32, u32, P, P]),
        "or_renorm_decode": (i32, [P, P, P]),
        "or_interleaved_encode": (i64, [P, u64, P, u32, u32, P, P, P, P]),
        "or_interleaved_decode": (i32, [P, u64, P, u64, P, u32, u32, P]),
        "or_backward_scan": (i32, [P, u64, u32, P, P, P]),
        "or_heuristic": (i64, [i64, i64, i64]),
        "or_choose_splits": (i64, [P, u64, u64, u32, u32, P]),
        "or_choose_splits_ex": (i64, [P, u64, u64, u32, u32, u32, P]),
        "or_recoil_encode_ex": (i32, [P, u64, P, u32, u32, u32, u32, P, P]),
        "or_pack_series": (u64, [P, u64, i32, u32, P, u64]),
        "or_unpack_series": (i64, [P, u64, u64, u64, i32, u32, P]),
        "or_decode_from": (i32, [P, u64, P, u32, u32, u64, i64, i64, P, P, u64, u64, P, P, P]),
        "or_recoil_encode": (i32, [P, u64, P, u32, u32, u32, P, P]),
        "or_combine": (i32, [P, u64, u32, P, P]),
        "or_container_info": (i32, [P, u64, P]),
        "or_container_points": (i32, [P, u64, P, P, P, P]),
        "or_recoil_decode": (i32, [P, u64, P]),
        "or_recoil_decode_task": (i32, [P, u64, u32, P, P, P]),
        "or_recoil_decode_tasks": (i32, [P, u64, P, u32, P, P]),
        "or_open": (i32, [P, u64, P]),
        "or_opened_decode_tasks": (i32, [P, P, u32, P, P]),
        "or_close": (None, [P]),
        "or_partitioned_encode": (i32, [P, u64, P, u32, u32, u32, P, P]),
        "or_partitioned_decode": (i32, [P, u64, P]),
        "or_quantize": (i32, [P, u32, u32, P]),
        "or_ad_interleaved_encode": (i64, [P, u64, P, u32, P, P, P, u32, u32, P, P, P]),
        "or_ad_interleaved_decode": (i32, [P, u64, P, u64, P, u32, P, P, P, u32, u32, P]),
        "or_ad_decode_from": (i32, [P, P, u32, P, P, P, u32, u32, u64, i64, i64, P, P, u64, u64, P]),
        "or_ad_recoil_encode": (i32, [P, u64, P, u32, P, P, P, u32, u32, u32, P, P]),
        "or_ad_recoil_decode": (i32, [P, u64, P, P]),
        "or_ad_recoil_decode_task": (i32, [P, u64, P, u32, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def _u8(buf) -> np.ndarray:
    if isinstance(buf, np.ndarray):
        return np.ascontiguousarray(buf, dtype=np.uint8)
    return np.frombuffer(bytes(buf), dtype=np.uint8)


def _check(rc):
    if rc < 0:
        raise OracleError(int(rc))
    return rc


def _freqs(f) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(f, dtype=np.uint32).reshape(256))


# --- model / single-lane primitives -------------------------------------------------

def build_model(hist, n: int) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(hist, dtype=np.uint64).reshape(256))
    f = np.zeros(256, dtype=np.uint32)
    _check(_load().or_build_model(h.ctypes.data, n, f.ctypes.data))
    return f


def cdf(f) -> np.ndarray:
    f = _freqs(f).astype(np.int64)
    return np.concatenate([[0], np.cumsum(f)[:-1]]).astype(np.uint32)


def encode_step(x: int, f: int, F: int, n: int) -> int:
    return int(_load().or_encode_step(x, f, F, n))


def decode_step(x: int, f, n: int) -> tuple[int, int]:
    s, xp = ctypes.c_uint32(), ctypes.c_uint32()
    _check(_load().or_decode_step(x, _freqs(f).ctypes.data, n, ctypes.byref(s), ctypes.byref(xp)))
    return s.value, xp.value


def renorm_encode(x: int, f_next: int, n: int):
    xv = ctypes.c_uint64(x)
    words = np.zeros(8, dtype=np.uint16)
    p = ctypes.c_uint64(0)
    steps = _load().or_renorm_encode(ctypes.byref(xv), f_next, n, words.ctypes.data, ctypes.byref(p))
    return xv.value, [int(w) for w in words[: p.value]], steps


def renorm_decode(x: int, words):
    xv = ctypes.c_uint64(x)
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint16))
    p = ctypes.c_int64(len(w) - 1)
    steps = _check(_load().or_renorm_decode(ctypes.byref(xv), _ptr(w), ctypes.byref(p)))
    return xv.value, steps, p.value


# --- interleaved codec ----------------------------------------------------------------

def interleaved_encode(sym, f, n: int, W: int = 32):
    """-> (words u16[B], final u32[W], events (structured), max_renorm_steps)"""
    s = _u8(sym)
    N = s.size
    words = np.zeros(N + 1, dtype=np.uint16)
    final = np.zeros(W, dtype=np.uint32)
    ev = np.zeros(N + 1, dtype=EVENT_DTYPE)
    steps = ctypes.c_uint64(0)
    B = _check(_load().or_interleaved_encode(_ptr(s), N, _freqs(f).ctypes.data, n, W, words.ctypes.data,
                                             final.ctypes.data, ev.ctypes.data, ctypes.byref(steps)))
    return words[:B].copy(), final, ev[:B].copy(), steps.value


def interleaved_decode(words, final, N: int, f, n: int, W: int = 32) -> np.ndarray:
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint16))
    fin = np.ascontiguousarray(np.asarray(final, dtype=np.uint32))
    out = np.zeros(N, dtype=np.uint8)
    _check(_load().or_interleaved_decode(_ptr(w), w.size, fin.ctypes.data, N, _freqs(f).ctypes.data, n, W,
                                         _ptr(out)))
    return out


def backward_scan(events, e: int, W: int):
    """-> None if infeasible, else (states[W], idx[W], sync_start)"""
    ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    st = np.zeros(W, dtype=np.uint32)
    ai = np.zeros(W, dtype=np.int64)
    ss = ctypes.c_int64(0)
    ok = _load().or_backward_scan(ev.ctypes.data, e, W, st.ctypes.data, ai.ctypes.data, ctypes.byref(ss))
    return (st, ai, ss.value) if ok else None


def heuristic(t: int, ts: int, T: int) -> int:
    return int(_load().or_heuristic(t, ts, T))


SPLIT_PRINTED_T = 1  # or_choose_splits_ex flag: T = ceil(N/M) as printed, not reading Z10''s T_m


def choose_splits(events, N: int, W: int, M: int, printed_T: bool = False) -> np.ndarray:
    ev = np.ascontiguousarray(events, dtype=EVENT_DTYPE)
    chosen = np.zeros(max(M, 1), dtype=np.uint64)
    k = _check(_load().or_choose_splits_ex(_ptr(ev), ev.size, N, W, M, SPLIT_PRINTED_T if printed_T else 0,
                                           chosen.ctypes.data))
    return chosen[:k].copy()


def pack_series(values, signed: bool, field_bits: int) -> tuple[bytes, int]:
    v = np.ascontiguousarray(np.asarray(values, dtype=np.int64))
    buf = np.zeros(8 + v.size * 9, dtype=np.uint8)
    bits = _load().or_pack_series(_ptr(v), v.size, int(signed), field_bits, buf.ctypes.data, 0)
    return bytes(buf[: (bits + 7) // 8]), int(bits)


def unpack_series(data: bytes, count: int, signed: bool, field_bits: int):
    b = np.frombuffer(bytes(data) + b"\0", dtype=np.uint8).copy()
    v = np.zeros(max(count, 1), dtype=np.int64)
    bits = _check(_load().or_unpack_series(b.ctypes.data, 8 * len(data), 0, count, int(signed), field_bits,
                                           v.ctypes.data))
    return [int(x) for x in v[:count]], int(bits)


def decode_from(words, f, n: int, W: int, N: int, cursor0: int, start_group: int, init_state, init_group,
                commit_lo: int, commit_hi: int, want_produced: bool = False):
    w = np.ascontiguousarray(np.asarray(words, dtype=np.uint16))
    st = np.ascontiguousarray(np.asarray(init_state, dtype=np.uint32))
    ig = np.ascontiguousarray(np.asarray(init_group, dtype=np.int64))
    out = np.zeros(max(N, 1), dtype=np.uint8)
    prod = np.zeros(max(N, 1), dtype=np.uint8)
    cend = ctypes.c_int64(0)
    rc = _load().or_decode_from(_ptr(w), w.size, _freqs(f).ctypes.data, n, W, N, cursor0, start_group,
                                st.ctypes.data, ig.ctypes.data, commit_lo, commit_hi, out.ctypes.data,
                                prod.ctypes.data if want_produced else None, ctypes.byref(cend))
    return rc, out[:N], (prod[:N].astype(bool) if want_produced else None), cend.value


# --- containers ---------------------------------------------------------------------

def _sized_call(fn, *args) -> bytes:
    ln = ctypes.c_uint64(0)
    _check(fn(*args, None, ctypes.byref(ln)))
    out = np.zeros(ln.value, dtype=np.uint8)
    _check(fn(*args, out.ctypes.data, ctypes.byref(ln)))
    return out[: ln.value].tobytes()


def recoil_encode(sym, f, n: int, M: int, W: int = 32, printed_T: bool = False) -> bytes:
    s = _u8(sym)
    return _sized_call(_load().or_recoil_encode_ex, _ptr(s), s.size, _freqs(f).ctypes.data, n, W, M,
                       SPLIT_PRINTED_T if printed_T else 0)


def combine(container: bytes, target: int) -> bytes:
    c = _u8(container)
    return _sized_call(_load().or_combine, c.ctypes.data, c.size, target)


def container_info(container: bytes) -> dict:
    c = _u8(container)
    info = np.zeros(8, dtype=np.uint64)
    _check(_load().or_container_info(c.ctypes.data, c.size, info.ctypes.data))
    keys = ["N", "B", "M", "n", "W", "header_model_bytes", "meta_bytes", "word_bytes"]
    return {k: int(v) for k, v in zip(keys, info)}


def container_points(container: bytes):
    info = container_info(container)
    P = info["M"] - 1
    c = _u8(container)
    arrs = [np.zeros(max(P, 1), dtype=np.uint64) for _ in range(4)]
    _check(_load().or_container_points(c.ctypes.data, c.size, *[a.ctypes.data for a in arrs]))
    return {k: a[:P].copy() for k, a in zip(["offset", "maxg", "sync_start", "bidx"], arrs)}


def recoil_decode(container: bytes) -> np.ndarray:
    c = _u8(container)
    N = container_info(container)["N"]
    out = np.zeros(max(N, 1), dtype=np.uint8)
    _check(_load().or_recoil_decode(c.ctypes.data, c.size, out.ctypes.data))
    return out[:N]


def recoil_decode_task(container: bytes, task: int, out: np.ndarray | None = None):
    """Decode one task into out (length N); returns (out, lo, hi)."""
    c = _u8(container)
    N = container_info(container)["N"]
    if out is None:
        out = np.zeros(max(N, 1), dtype=np.uint8)
    lo, hi = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _check(_load().or_recoil_decode_task(c.ctypes.data, c.size, task, out.ctypes.data, ctypes.byref(lo),
                                         ctypes.byref(hi)))
    return out, lo.value, hi.value


def recoil_decode_tasks(container: bytes, tasks, out: np.ndarray | None = None):
    """Decode a list of tasks with one container parse; returns (out, committed symbols)."""
    c = _u8(container)
    N = container_info(container)["N"]
    if out is None:
        out = np.zeros(max(N, 1), dtype=np.uint8)
    t = np.ascontiguousarray(np.asarray(tasks, dtype=np.uint32))
    n = ctypes.c_uint64(0)
    _check(_load().or_recoil_decode_tasks(c.ctypes.data, c.size, _ptr(t), t.size, out.ctypes.data, ctypes.byref(n)))
    return out, n.value


class Opened:
    """A container parsed once (or_open) for repeated task decodes; the parse stays
    outside any timed region that uses decode_tasks."""

    def __init__(self, container: bytes):
        self._c = _u8(container)  # or_open keeps pointers into the container bytes
        self.info = container_info(container)
        self.h = ctypes.c_void_p()
        _check(_load().or_open(self._c.ctypes.data, self._c.size, ctypes.byref(self.h)))

    def decode_tasks(self, tasks, out: np.ndarray):
        t = np.ascontiguousarray(np.asarray(tasks, dtype=np.uint32))
        n = ctypes.c_uint64(0)
        _check(_load().or_opened_decode_tasks(self.h, _ptr(t), t.size, out.ctypes.data, ctypes.byref(n)))
        return n.value

    def close(self):
        if self.h:
            _load().or_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def partitioned_encode(sym, f, n: int, P: int, W: int = 32) -> bytes:
    s = _u8(sym)
    return _sized_call(_load().or_partitioned_encode, _ptr(s), s.size, _freqs(f).ctypes.data, n, W, P)


def partitioned_decode(container: bytes) -> np.ndarray:
    c = _u8(container)
    N = int.from_bytes(bytes(c[12:20]), "little")
    out = np.zeros(max(N, 1), dtype=np.uint8)
    _check(_load().or_partitioned_decode(c.ctypes.data, c.size, out.ctypes.data))
    return out[:N]


# --- adaptive coding: index-keyed models, 16-bit symbols (P:227 (3)) ---------

def quantize(hist, n: int) -> np.ndarray:
    """Reading Z19's quantiser over any number of entries (build_model = 256 entries)."""
    h = np.ascontiguousarray(np.asarray(hist, dtype=np.uint64))
    f = np.zeros(h.size, dtype=np.uint32)
    _check(_load().or_quantize(h.ctypes.data, h.size, n, f.ctypes.data))
    return f


def _models(models):
    base = np.ascontiguousarray(np.asarray(models["base"], dtype=np.uint32))
    ln = np.ascontiguousarray(np.asarray(models["len"], dtype=np.uint32))
    f = np.ascontiguousarray(np.asarray(models["f"], dtype=np.uint32))
    assert base.size == ln.size and f.size == int(ln.sum())
    return base, ln, f


def _u16(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint16))


def _mid(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8))


def ad_interleaved_encode(sym, mid, models, n: int, W: int = 32):
    """-> (words u16[B], final u32[W], events)"""
    s, m = _u16(sym), _mid(mid)
    base, ln, f = _models(models)
    N = s.size
    words = np.zeros(4 * N + 8, dtype=np.uint16)
    final = np.zeros(W, dtype=np.uint32)
    ev = np.zeros(4 * N + 8, dtype=EVENT_DTYPE)
    B = _check(_load().or_ad_interleaved_encode(_ptr(s), N, _ptr(m), base.size, base.ctypes.data, ln.ctypes.data,
                                                f.ctypes.data, n, W, words.ctypes.data, final.ctypes.data,
                                                ev.ctypes.data))
    return words[:B].copy(), final, ev[:B].copy()


def ad_interleaved_decode(words, final, N: int, mid, models, n: int, W: int = 32) -> np.ndarray:
    w = _u16(words)
    fin = np.ascontiguousarray(np.asarray(final, dtype=np.uint32))
    m = _mid(mid)
    base, ln, f = _models(models)
    out = np.zeros(max(N, 1), dtype=np.uint16)
    _check(_load().or_ad_interleaved_decode(_ptr(w), w.size, fin.ctypes.data, N, _ptr(m), base.size, base.ctypes.data,
                                            ln.ctypes.data, f.ctypes.data, n, W, out.ctypes.data))
    return out[:N]


def ad_decode_from(words, mid, models, n: int, W: int, N: int, cursor0: int, start_group: int, init_state,
                   init_group, commit_lo: int, commit_hi: int):
    w = _u16(words)
    m = _mid(mid)
    base, ln, f = _models(models)
    st = np.ascontiguousarray(np.asarray(init_state, dtype=np.uint32))
    ig = np.ascontiguousarray(np.asarray(init_group, dtype=np.int64))
    out = np.zeros(max(N, 1), dtype=np.uint16)
    rc = _load().or_ad_decode_from(_ptr(w), _ptr(m), base.size, base.ctypes.data, ln.ctypes.data, f.ctypes.data, n, W,
                                   N, cursor0, start_group, st.ctypes.data, ig.ctypes.data, commit_lo, commit_hi,
                                   out.ctypes.data)
    return rc, out[:N]


def ad_recoil_encode(sym, mid, models, n: int, M: int, W: int = 32) -> bytes:
    s, m = _u16(sym), _mid(mid)
    base, ln, f = _models(models)
    return _sized_call(_load().or_ad_recoil_encode, _ptr(s), s.size, _ptr(m), base.size, base.ctypes.data,
                       ln.ctypes.data, f.ctypes.data, n, W, M)


def ad_recoil_decode(container: bytes, mid) -> np.ndarray:
    c = _u8(container)
    m = _mid(mid)
    N = container_info(container)["N"]
    out = np.zeros(max(N, 1), dtype=np.uint16)
    _check(_load().or_ad_recoil_decode(c.ctypes.data, c.size, _ptr(m), out.ctypes.data))
    return out[:N]


def ad_recoil_decode_task(container: bytes, mid, task: int, out: np.ndarray | None = None):
    c = _u8(container)
    m = _mid(mid)
    N = container_info(container)["N"]
    if out is None:
        out = np.zeros(max(N, 1), dtype=np.uint16)
    lo, hi = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _check(_load().or_ad_recoil_decode_task(c.ctypes.data, c.size, _ptr(m), task, out.ctypes.data,
                                            ctypes.byref(lo), ctypes.byref(hi)))
    return out, lo.value, hi.value
