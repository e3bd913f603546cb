"""Thin ctypes binding of librecoil.so (include/recoil.h).  Argument marshalling only:
every step of the decode path runs in the library (host C++ for encode/metadata,
sm_100a CUDA kernels for decode).  There is no Python or CPU fallback: if the
library is missing or fails to load, every call raises.

Function names equal the C ABI names.  Host buffers are numpy arrays / bytes;
device buffers are torch CUDA tensors (PyTorch supplies device memory and
streams only).  Errors raise ``RecoilError`` carrying the RECOIL_E_* code.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RECOIL_LIB") or os.path.join(_PKG, "librecoil.so")  # RECOIL_LIB: experiment builds
_lib = None

RECOIL_OK = 0
ERRORS = {
    -1: "RECOIL_E_ARG", -2: "RECOIL_E_EMPTY", -3: "RECOIL_E_ALPHABET", -4: "RECOIL_E_ZERO_FREQ",
    -5: "RECOIL_E_OVERFLOW", -6: "RECOIL_E_BAD_MAGIC", -7: "RECOIL_E_VERSION", -8: "RECOIL_E_TRUNCATED",
    -9: "RECOIL_E_INCONSISTENT", -10: "RECOIL_E_UNDERFLOW", -11: "RECOIL_E_SYNC", -12: "RECOIL_E_CUDA",
    -13: "RECOIL_E_NOMEM", -14: "RECOIL_E_BUFFER", -15: "RECOIL_E_UNSUPPORTED",
}
globals().update({v: k for k, v in ERRORS.items()})

EXPORTS = [
    "recoil_strerror", "recoil_build_model", "recoil_encode", "recoil_combine_splits", "recoil_inspect",
    "recoil_partitioned_encode", "recoil_decoder_create", "recoil_decoder_plan", "recoil_decoder_upload",
    "recoil_decode", "recoil_decoder_status", "recoil_decoder_launches", "recoil_decoder_destroy",
    "recoil_decode_occupancy", "recoil_shard_plan", "recoil_decode_cpu", "recoil_decode_cpu_ex", "recoil_cpu_simd",
    "recoil_pipeline_create", "recoil_pipeline_device_bytes", "recoil_pipeline_run", "recoil_pipeline_status",
    "recoil_pipeline_launches", "recoil_pipeline_destroy", "recoil_quantize", "recoil_encode_adaptive",
    "recoil_decode_adaptive", "recoil_decode_occupancy_adaptive", "recoil_decoder_create_subset",
    "recoil_decoder_create_grouped", "recoil_decoder_create_for_device", "recoil_pipeline_run_at", "recoil_pipeline_span", "recoil_multi_plan",
    "recoil_multi_decode", "recoil_multi_nccl_available", "recoil_device_decoder_create",
    "recoil_device_decoder_plan", "recoil_device_upload", "recoil_device_decode", "recoil_device_decoder_status",
    "recoil_device_decoder_launches", "recoil_device_decoder_destroy", "recoil_device_combine_plan",
    "recoil_device_combine", "recoil_device_decoder_create_range", "recoil_device_decoder_span",
]


class RecoilError(RuntimeError):
    def __init__(self, rc: int, what: str = ""):
        name = ERRORS.get(rc, str(rc))
        super().__init__(f"{what}: {name}" if what else name)
        self.rc = rc


class recoil_info(ctypes.Structure):
    _fields_ = [("n_symbols", ctypes.c_uint64), ("n_words", ctypes.c_uint64), ("n_splits", ctypes.c_uint32),
                ("prob_bits", ctypes.c_uint32), ("lanes", ctypes.c_uint32), ("partitioned", ctypes.c_uint32),
                ("header_bytes", ctypes.c_uint64), ("meta_bytes", ctypes.c_uint64),
                ("word_bytes", ctypes.c_uint64), ("total_bytes", ctypes.c_uint64),
                ("symbol_bits", ctypes.c_uint32), ("n_models", ctypes.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class recoil_device_plan(ctypes.Structure):
    _fields_ = [("container_offset", ctypes.c_uint64), ("buffer_bytes", ctypes.c_uint64),
                ("workspace_bytes", ctypes.c_uint64), ("out_count", ctypes.c_uint64), ("n_symbols", ctypes.c_uint64),
                ("n_tasks", ctypes.c_uint32), ("prob_bits", ctypes.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class recoil_plan(ctypes.Structure):
    _fields_ = [("task_begin", ctypes.c_uint64), ("task_end", ctypes.c_uint64), ("n_tasks", ctypes.c_uint32),
                ("prob_bits", ctypes.c_uint32), ("word_lo", ctypes.c_uint64), ("word_count", ctypes.c_uint64),
                ("out_lo", ctypes.c_uint64), ("out_hi", ctypes.c_uint64), ("out_base", ctypes.c_uint64),
                ("out_count", ctypes.c_uint64), ("workspace_bytes", ctypes.c_uint64),
                ("upload_bytes", ctypes.c_uint64), ("symbol_bytes", ctypes.c_uint32), ("n_models", ctypes.c_uint32),
                ("coarse_bits", ctypes.c_uint32), ("warps_per_block", ctypes.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def load(path: str = LIB_PATH):
    """Load librecoil.so; raises if it is missing (build with __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"librecoil.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    P, u32, u64, i32 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
    sig = {
        "recoil_strerror": (ctypes.c_char_p, [i32]),
        "recoil_build_model": (i32, [P, u32, P]),
        "recoil_encode": (i32, [P, u64, P, u32, u32, P, P]),
        "recoil_combine_splits": (i32, [P, u64, u32, P, P]),
        "recoil_inspect": (i32, [P, u64, P]),
        "recoil_partitioned_encode": (i32, [P, u64, P, u32, u32, P, P]),
        "recoil_decoder_create": (i32, [P, u64, u64, u64, P]),
        "recoil_decoder_plan": (i32, [P, P]),
        "recoil_decoder_upload": (i32, [P, P, P, P]),
        "recoil_decode": (i32, [P, P, P, P, P]),
        "recoil_decoder_status": (i32, [P, P, P, P]),
        "recoil_decoder_launches": (i32, [P]),
        "recoil_decoder_destroy": (None, [P]),
        "recoil_decode_occupancy": (i32, [i32, u32, P, P]),
        "recoil_shard_plan": (i32, [P, u64, u32, P]),
        "recoil_decode_cpu": (i32, [P, u64, P, u32]),
        "recoil_decode_cpu_ex": (i32, [P, u64, P, u32, u32]),
        "recoil_cpu_simd": (i32, []),
        "recoil_pipeline_create": (i32, [P, u64, u64, u64, u32, P]),
        "recoil_pipeline_device_bytes": (i32, [P, u32, P]),
        "recoil_pipeline_run": (i32, [P, P, P, P, u32]),
        "recoil_pipeline_status": (i32, [P, P, u32, P]),
        "recoil_pipeline_launches": (i32, [P]),
        "recoil_pipeline_destroy": (None, [P]),
        "recoil_quantize": (i32, [P, u32, u32, P]),
        "recoil_encode_adaptive": (i32, [P, u64, P, u32, P, P, P, u32, u32, P, P]),
        "recoil_decode_adaptive": (i32, [P, P, P, P, P, P]),
        "recoil_decode_occupancy_adaptive": (i32, [i32, u32, u64, P, P]),
        "recoil_decoder_create_subset": (i32, [P, u64, u32, u64, u64, P]),
        "recoil_decoder_create_grouped": (i32, [P, u64, u32, P, P, P]),
        "recoil_pipeline_run_at": (i32, [P, P, P, u64, P, u32]),
        "recoil_decoder_create_for_device": (i32, [P, u64, i32, u32, P]),
        "recoil_pipeline_span": (i32, [P, P, P]),
        "recoil_multi_plan": (i32, [P, u64, u32, P]),
        "recoil_multi_decode": (i32, [P, u64, u32, P, P, i32, P, P]),
        "recoil_multi_nccl_available": (i32, []),
        "recoil_device_decoder_create": (i32, [P, u64, u64, P]),
        "recoil_device_decoder_create_range": (i32, [P, u64, u64, u64, u64, P]),
        "recoil_device_decoder_span": (i32, [P, P, P, P, P]),
        "recoil_device_decoder_plan": (i32, [P, P]),
        "recoil_device_upload": (i32, [P, P, P, P]),
        "recoil_device_decode": (i32, [P, P, P, P, P]),
        "recoil_device_decoder_status": (i32, [P, P, P, P]),
        "recoil_device_decoder_launches": (i32, [P]),
        "recoil_device_decoder_destroy": (None, [P]),
        "recoil_device_combine_plan": (i32, [P, u64, u64, u32, P, P]),
        "recoil_device_combine": (i32, [P, u64, P, u64, u32, P, u64, P, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int, what: str = "") -> int:
    if rc < 0:
        raise RecoilError(rc, what)
    return rc


def _u8(buf) -> np.ndarray:
    if isinstance(buf, np.ndarray):
        return np.ascontiguousarray(buf.reshape(-1).view(np.uint8))
    return np.frombuffer(memoryview(buf), dtype=np.uint8)


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def _freqs(f) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(f, dtype=np.uint32).reshape(256))


def recoil_strerror(rc: int) -> str:
    return load().recoil_strerror(rc).decode()


def recoil_build_model(hist, prob_bits: int) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(hist, dtype=np.uint64).reshape(256))
    f = np.zeros(256, dtype=np.uint32)
    _check(load().recoil_build_model(h.ctypes.data, prob_bits, f.ctypes.data), "recoil_build_model")
    return f


def _sized(fn, what, *args) -> np.ndarray:
    n = ctypes.c_uint64(0)
    _check(fn(*args, None, ctypes.byref(n)), what)
    out = np.empty(n.value, dtype=np.uint8)
    rc = fn(*args, out.ctypes.data, ctypes.byref(n))
    if rc == RECOIL_E_BUFFER:
        out = np.empty(n.value, dtype=np.uint8)
        rc = fn(*args, out.ctypes.data, ctypes.byref(n))
    _check(rc, what)
    return out[: n.value]


def recoil_encode(symbols, freqs, prob_bits: int, n_splits: int) -> np.ndarray:
    """-> container bytes (numpy uint8)."""
    s = _u8(symbols)
    return _sized(load().recoil_encode, "recoil_encode", _ptr(s), s.size, _freqs(freqs).ctypes.data, prob_bits,
                  n_splits)


def recoil_partitioned_encode(symbols, freqs, prob_bits: int, n_partitions: int) -> np.ndarray:
    s = _u8(symbols)
    return _sized(load().recoil_partitioned_encode, "recoil_partitioned_encode", _ptr(s), s.size,
                  _freqs(freqs).ctypes.data, prob_bits, n_partitions)


def recoil_combine_splits(container, target_splits: int) -> np.ndarray:
    c = _u8(container)
    return _sized(load().recoil_combine_splits, "recoil_combine_splits", c.ctypes.data, c.size, target_splits)


def recoil_inspect(container) -> dict:
    c = _u8(container)
    info = recoil_info()
    _check(load().recoil_inspect(c.ctypes.data, c.size, ctypes.byref(info)), "recoil_inspect")
    return info.as_dict()


def recoil_shard_plan(container, n_shards: int) -> list[int]:
    c = _u8(container)
    b = np.zeros(n_shards + 1, dtype=np.uint64)
    _check(load().recoil_shard_plan(c.ctypes.data, c.size, n_shards, b.ctypes.data), "recoil_shard_plan")
    return [int(x) for x in b]


def recoil_decode_cpu(container, threads: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    c = _u8(container)
    N = recoil_inspect(c)["n_symbols"]
    if out is None:
        out = np.empty(N, dtype=np.uint8)
    _check(load().recoil_decode_cpu(c.ctypes.data, c.size, _ptr(out), threads), "recoil_decode_cpu")
    return out


RECOIL_CPU_SCALAR = 1
RECOIL_CPU_AVX2 = 2


def recoil_decode_cpu_ex(container, threads: int = 0, flags: int = 0, out: np.ndarray | None = None) -> np.ndarray:
    c = _u8(container)
    N = recoil_inspect(c)["n_symbols"]
    if out is None:
        out = np.empty(N, dtype=np.uint8)
    _check(load().recoil_decode_cpu_ex(c.ctypes.data, c.size, _ptr(out), threads, flags), "recoil_decode_cpu_ex")
    return out


def recoil_cpu_simd() -> int:
    """2 = AVX-512, 1 = AVX2, 0 = scalar (the task decoder recoil_decode_cpu uses here)."""
    return int(load().recoil_cpu_simd())


def recoil_cpu_isa() -> str:
    return {2: "avx512", 1: "avx2", 0: "scalar"}[recoil_cpu_simd()]


def recoil_decode_occupancy(device: int, prob_bits: int) -> tuple[int, int]:
    w, s = ctypes.c_int(0), ctypes.c_int(0)
    _check(load().recoil_decode_occupancy(device, prob_bits, ctypes.byref(w), ctypes.byref(s)),
           "recoil_decode_occupancy")
    return w.value, s.value


# --- decoder handle ---------------------------------------------------------------------

def recoil_decoder_create(container, task_begin: int = 0, task_end: int = (1 << 64) - 1) -> ctypes.c_void_p:
    c = _u8(container)
    h = ctypes.c_void_p()
    _check(load().recoil_decoder_create(c.ctypes.data, c.size, task_begin, task_end, ctypes.byref(h)),
           "recoil_decoder_create")
    return h


def recoil_decoder_create_subset(container, target_splits: int, task_begin: int = 0,
                                 task_end: int = (1 << 64) - 1) -> ctypes.c_void_p:
    c = _u8(container)
    h = ctypes.c_void_p()
    _check(load().recoil_decoder_create_subset(c.ctypes.data, c.size, target_splits, task_begin, task_end,
                                               ctypes.byref(h)), "recoil_decoder_create_subset")
    return h


def recoil_decoder_create_for_device(container, device: int = 0, waves_x100: int = 0) -> ctypes.c_void_p:
    c = _u8(container)
    h = ctypes.c_void_p()
    _check(load().recoil_decoder_create_for_device(c.ctypes.data, c.size, device, waves_x100, ctypes.byref(h)),
           "recoil_decoder_create_for_device")
    return h


def recoil_decoder_create_grouped(container, run_tasks, run_splits) -> ctypes.c_void_p:
    """Tasks in stream order: run_tasks[r] tasks of run_splits[r] encoder splits each, the last task
    takes the rest."""
    c = _u8(container)
    rt = np.ascontiguousarray(np.asarray(run_tasks, dtype=np.uint32))
    rs = np.ascontiguousarray(np.asarray(run_splits, dtype=np.uint32))
    if rt.size != rs.size:
        raise ValueError("run_tasks and run_splits differ in length")
    h = ctypes.c_void_p()
    _check(load().recoil_decoder_create_grouped(c.ctypes.data, c.size, rt.size, _ptr(rt), _ptr(rs),
                                                ctypes.byref(h)), "recoil_decoder_create_grouped")
    return h


def recoil_decoder_plan(handle) -> dict:
    p = recoil_plan()
    _check(load().recoil_decoder_plan(handle, ctypes.byref(p)), "recoil_decoder_plan")
    return p.as_dict()


def recoil_decoder_upload(handle, d_workspace: int, d_words: int, stream: int) -> None:
    _check(load().recoil_decoder_upload(handle, d_workspace, d_words, stream), "recoil_decoder_upload")


def recoil_decode(handle, d_workspace: int, d_words: int, d_out: int, stream: int) -> None:
    _check(load().recoil_decode(handle, d_workspace, d_words, d_out, stream), "recoil_decode")


def recoil_decoder_status(handle, d_workspace: int, stream: int) -> tuple[int, int | None]:
    bad = ctypes.c_uint64(0)
    rc = load().recoil_decoder_status(handle, d_workspace, stream, ctypes.byref(bad))
    return rc, (None if bad.value == (1 << 64) - 1 else bad.value)


def recoil_decoder_launches(handle) -> int:
    return _check(load().recoil_decoder_launches(handle), "recoil_decoder_launches")


def recoil_decoder_destroy(handle) -> None:
    if handle:
        load().recoil_decoder_destroy(handle)


def recoil_quantize(hist, prob_bits: int) -> np.ndarray:
    h = np.ascontiguousarray(np.asarray(hist, dtype=np.uint64))
    f = np.zeros(h.size, dtype=np.uint32)
    _check(load().recoil_quantize(h.ctypes.data, h.size, prob_bits, f.ctypes.data), "recoil_quantize")
    return f


def recoil_encode_adaptive(symbols, model_ids, models, prob_bits: int, n_splits: int) -> np.ndarray:
    """models: {"base": u32[K], "len": u32[K], "f": u32[sum len]}"""
    s = np.ascontiguousarray(np.asarray(symbols, dtype=np.uint16))
    m = np.ascontiguousarray(np.asarray(model_ids, dtype=np.uint8))
    base = np.ascontiguousarray(np.asarray(models["base"], dtype=np.uint32))
    ln = np.ascontiguousarray(np.asarray(models["len"], dtype=np.uint32))
    f = np.ascontiguousarray(np.asarray(models["f"], dtype=np.uint32))
    return _sized(load().recoil_encode_adaptive, "recoil_encode_adaptive", _ptr(s), s.size, _ptr(m), base.size,
                  base.ctypes.data, ln.ctypes.data, f.ctypes.data, prob_bits, n_splits)


def recoil_decode_adaptive(handle, d_workspace: int, d_words: int, d_model_ids: int, d_out: int, stream: int) -> None:
    _check(load().recoil_decode_adaptive(handle, d_workspace, d_words, d_model_ids, d_out, stream),
           "recoil_decode_adaptive")


def recoil_decode_occupancy_adaptive(device: int, n_models: int, n_entries: int) -> tuple[int, int]:
    """(resident warps per SM, SMs) of the adaptive kernel for n_models models with n_entries
    table entries in total (an upper bound such as the model set's total value count is fine)."""
    w, s = ctypes.c_int(0), ctypes.c_int(0)
    _check(load().recoil_decode_occupancy_adaptive(device, n_models, n_entries, ctypes.byref(w), ctypes.byref(s)),
           "recoil_decode_occupancy_adaptive")
    return w.value, s.value


class GpuDecoder:
    """Owns a decoder handle plus the torch device buffers of its plan.

    ``container`` must stay alive as long as this object (the handle points into it).
    """

    def __init__(self, container, device: int = 0, task_begin: int = 0, task_end: int = (1 << 64) - 1,
                 stream=None, subset: int | None = None, grouped=None, for_device: bool = False):
        import torch
        self.container = _u8(container)
        self.device = torch.device("cuda", device)
        if for_device:  # decoder-adaptive: combine in place to this GPU's parallelism
            self.handle = recoil_decoder_create_for_device(self.container, device)
        elif grouped is not None:  # (run_tasks, run_splits): recoil_decoder_create_grouped
            self.handle = recoil_decoder_create_grouped(self.container, *grouped)
        else:
            self.handle = (recoil_decoder_create(self.container, task_begin, task_end) if subset is None else
                           recoil_decoder_create_subset(self.container, subset, task_begin, task_end))
        self.plan = recoil_decoder_plan(self.handle)
        p = self.plan
        self.stream = stream or torch.cuda.current_stream(self.device)
        self.workspace = torch.empty(max(p["workspace_bytes"], 16), dtype=torch.uint8, device=self.device)
        self.words = torch.empty(max(p["word_count"], 1), dtype=torch.int16, device=self.device)
        self.adaptive = p["symbol_bytes"] == 2
        self.out = torch.empty(max(p["out_count"], 16), dtype=torch.int16 if self.adaptive else torch.uint8,
                               device=self.device)
        self.model_ids = None  # adaptive: device tensor of the stream's model ids (set_model_ids)

    def set_model_ids(self, model_ids) -> None:
        """Adaptive containers: the model id of every symbol of the stream (host or device)."""
        import torch
        t = torch.as_tensor(np.ascontiguousarray(model_ids, dtype=np.uint8)) if not torch.is_tensor(model_ids) \
            else model_ids
        n = t.numel()
        buf = torch.zeros(((n + 15) // 16) * 16 + 16, dtype=torch.uint8, device=self.device)
        buf[:n].copy_(t.reshape(-1).to(torch.uint8), non_blocking=False)
        self.model_ids = buf

    @property
    def stream_handle(self) -> int:
        return self.stream.cuda_stream

    def upload(self) -> None:
        recoil_decoder_upload(self.handle, self.workspace.data_ptr(), self.words.data_ptr(), self.stream_handle)

    def decode(self, out=None) -> None:
        o = self.out if out is None else out
        if self.adaptive:
            if self.model_ids is None:
                raise RuntimeError("adaptive container: call set_model_ids first")
            recoil_decode_adaptive(self.handle, self.workspace.data_ptr(), self.words.data_ptr(),
                                   self.model_ids.data_ptr(), o.data_ptr(), self.stream_handle)
            return
        recoil_decode(self.handle, self.workspace.data_ptr(), self.words.data_ptr(), o.data_ptr(),
                      self.stream_handle)

    def status(self) -> tuple[int, int | None]:
        return recoil_decoder_status(self.handle, self.workspace.data_ptr(), self.stream_handle)

    def output(self):
        """Committed symbols [out_lo, out_hi) as a device tensor view."""
        p = self.plan
        return self.out[p["out_lo"] - p["out_base"]: p["out_hi"] - p["out_base"]]

    def launches(self) -> int:
        return recoil_decoder_launches(self.handle)

    def close(self) -> None:
        recoil_decoder_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            if self.handle:
                self.close()
        except Exception:
            pass


def recoil_pipeline_create(container, n_chunks: int, task_begin: int = 0,
                           task_end: int = (1 << 64) - 1) -> ctypes.c_void_p:
    c = _u8(container)
    h = ctypes.c_void_p()
    _check(load().recoil_pipeline_create(c.ctypes.data, c.size, task_begin, task_end, n_chunks, ctypes.byref(h)),
           "recoil_pipeline_create")
    return h


def recoil_pipeline_device_bytes(handle, n_streams: int) -> int:
    b = ctypes.c_uint64(0)
    _check(load().recoil_pipeline_device_bytes(handle, n_streams, ctypes.byref(b)), "recoil_pipeline_device_bytes")
    return b.value


def _streams(streams):
    arr = (ctypes.c_void_p * len(streams))(*[s for s in streams])
    return arr, len(streams)


def recoil_pipeline_run(handle, d_scratch: int, host_out: int, streams) -> None:
    arr, n = _streams(streams)
    _check(load().recoil_pipeline_run(handle, d_scratch, host_out, arr, n), "recoil_pipeline_run")


def recoil_pipeline_run_at(handle, d_scratch: int, host_out: int, host_first: int, streams) -> None:
    arr, n = _streams(streams)
    _check(load().recoil_pipeline_run_at(handle, d_scratch, host_out, host_first, arr, n), "recoil_pipeline_run_at")


def recoil_pipeline_span(handle) -> tuple[int, int]:
    lo, hi = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _check(load().recoil_pipeline_span(handle, ctypes.byref(lo), ctypes.byref(hi)), "recoil_pipeline_span")
    return lo.value, hi.value


def recoil_pipeline_status(handle, streams) -> tuple[int, int | None]:
    arr, n = _streams(streams)
    bad = ctypes.c_uint64(0)
    rc = load().recoil_pipeline_status(handle, arr, n, ctypes.byref(bad))
    return rc, (None if bad.value == (1 << 64) - 1 else bad.value)


def recoil_pipeline_launches(handle) -> int:
    return _check(load().recoil_pipeline_launches(handle), "recoil_pipeline_launches")


def recoil_pipeline_destroy(handle) -> None:
    if handle:
        load().recoil_pipeline_destroy(handle)


class HostPipeline:
    """End-to-end host->host decode on one GPU (recoil_pipeline_*): owns the handle,
    the torch device scratch and the CUDA streams.  ``container`` should be pinned."""

    def __init__(self, container, device: int = 0, n_chunks: int = 8, n_streams: int = 3, task_begin: int = 0,
                 task_end: int = (1 << 64) - 1):
        import torch
        self.container = _u8(container)
        self.device = torch.device("cuda", device)
        self.handle = recoil_pipeline_create(self.container, n_chunks, task_begin, task_end)
        self.streams = [torch.cuda.Stream(self.device) for _ in range(n_streams)]
        self.scratch = torch.empty(max(recoil_pipeline_device_bytes(self.handle, n_streams), 256),
                                   dtype=torch.uint8, device=self.device)

    def run(self, host_out, host_first: int = 0) -> None:
        """host_out[i - host_first] receives symbol i of the pipeline's span (host_first = 0:
        a buffer of the whole stream; = span()[0]: a buffer of the span only)."""
        ptr = host_out.data_ptr() if hasattr(host_out, "data_ptr") else host_out.ctypes.data
        recoil_pipeline_run_at(self.handle, self.scratch.data_ptr(), ptr, host_first,
                               [s.cuda_stream for s in self.streams])

    def span(self) -> tuple[int, int]:
        return recoil_pipeline_span(self.handle)

    def status(self):
        return recoil_pipeline_status(self.handle, [s.cuda_stream for s in self.streams])

    def launches(self) -> int:
        return recoil_pipeline_launches(self.handle)

    def close(self) -> None:
        recoil_pipeline_destroy(self.handle)
        self.handle = None

    def __del__(self):
        try:
            if self.handle:
                self.close()
        except Exception:
            pass


def decode_gpu(container, device: int = 0):
    """Convenience: full decode on one GPU; returns the device tensor of N symbols
    (raises RecoilError on a device status error)."""
    dec = GpuDecoder(container, device)
    dec.upload()
    dec.decode()
    rc, bad = dec.status()
    if rc:
        raise RecoilError(rc, f"decode (task {bad})")
    out = dec.output().clone()
    dec.close()
    return out


# --- on-device metadata path (NEXT 2): the container goes to the GPU as it is -------------

class DeviceContainerDecoder:
    """recoil_device_*: the host reads the fixed header + model block only; the container is
    copied to the GPU unchanged and its split metadata decoded there (global series, record
    offsets, LUT, task heads), then the decode kernel runs.  Device buffers are torch tensors."""

    def __init__(self, container, device: int = 0, stream=None, task_begin: int = 0, task_end: int | None = None):
        import torch
        c = _u8(container)
        self.container = c
        self.device = torch.device("cuda", device)
        h = ctypes.c_void_p()
        te = (1 << 64) - 1 if task_end is None else task_end
        _check(load().recoil_device_decoder_create_range(c.ctypes.data, c.size, c.size, task_begin, te,
                                                         ctypes.byref(h)), "recoil_device_decoder_create_range")
        self.handle = h
        pl = recoil_device_plan()
        _check(load().recoil_device_decoder_plan(h, ctypes.byref(pl)), "recoil_device_decoder_plan")
        self.plan = pl.as_dict()
        self.stream = stream or torch.cuda.current_stream(self.device)
        self.buffer = torch.empty(self.plan["buffer_bytes"], dtype=torch.uint8, device=self.device)
        self.workspace = torch.empty(max(self.plan["workspace_bytes"], 256), dtype=torch.uint8, device=self.device)
        self.out = torch.empty(max(self.plan["out_count"], 16), dtype=torch.uint8, device=self.device)

    def upload(self, container=None) -> None:
        """H2D of the container bytes (pinned for an asynchronous copy) + zero padding."""
        c = self.container if container is None else container
        ptr = c.data_ptr() if hasattr(c, "data_ptr") else _u8(c).ctypes.data
        _check(load().recoil_device_upload(self.handle, ptr, self.buffer.data_ptr(), self.stream.cuda_stream),
               "recoil_device_upload")

    def decode(self) -> None:
        _check(load().recoil_device_decode(self.handle, self.buffer.data_ptr(), self.workspace.data_ptr(),
                                           self.out.data_ptr(), self.stream.cuda_stream), "recoil_device_decode")

    def status(self):
        bad = ctypes.c_uint64(0)
        rc = load().recoil_device_decoder_status(self.handle, self.workspace.data_ptr(), self.stream.cuda_stream,
                                                 ctypes.byref(bad))
        return rc, (None if bad.value == (1 << 64) - 1 else bad.value)

    def output(self):
        return self.out[:self.plan["n_symbols"]]

    def span(self) -> tuple[int, int]:
        """The committed symbol span [lo, hi) of this decoder's task range (after decode)."""
        lo, hi = ctypes.c_uint64(0), ctypes.c_uint64(0)
        _check(load().recoil_device_decoder_span(self.handle, self.workspace.data_ptr(), self.stream.cuda_stream,
                                                 ctypes.byref(lo), ctypes.byref(hi)), "recoil_device_decoder_span")
        return lo.value, hi.value

    def launches(self) -> int:
        return _check(load().recoil_device_decoder_launches(self.handle), "recoil_device_decoder_launches")

    def close(self) -> None:
        if self.handle:
            load().recoil_device_decoder_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def recoil_device_combine(container, d_in, target_splits: int, stream=None):
    """Combine on the GPU: d_in (torch uint8 tensor holding `container`) -> a new device tensor
    with the combined container (recoil_combine_splits(container, target_splits) byte for byte)."""
    import torch
    c = _u8(container)
    cap, wsb = ctypes.c_uint64(0), ctypes.c_uint64(0)
    _check(load().recoil_device_combine_plan(c.ctypes.data, c.size, c.size, target_splits, ctypes.byref(cap),
                                             ctypes.byref(wsb)), "recoil_device_combine_plan")
    out = torch.empty(cap.value, dtype=torch.uint8, device=d_in.device)
    ws = torch.empty(max(wsb.value, 256), dtype=torch.uint8, device=d_in.device)
    n = torch.zeros(1, dtype=torch.int64, device=d_in.device)
    st = stream or torch.cuda.current_stream(d_in.device)
    _check(load().recoil_device_combine(c.ctypes.data, c.size, d_in.data_ptr(), c.size, target_splits,
                                        out.data_ptr(), cap.value, ws.data_ptr(), n.data_ptr(), st.cuda_stream),
           "recoil_device_combine")
    st.synchronize()
    return out[:int(n.item())]


# --- multi-GPU (§8(e), row a10): optional gather of the shards' spans ----------------------

def recoil_multi_plan(container, n_dev: int) -> list[dict]:
    c = _u8(container)
    plans = (recoil_plan * n_dev)()
    _check(load().recoil_multi_plan(c.ctypes.data, c.size, n_dev, plans), "recoil_multi_plan")
    return [p.as_dict() for p in plans]


def recoil_multi_nccl_available() -> bool:
    return bool(load().recoil_multi_nccl_available())


def recoil_multi_decode(container, devices, d_outs, gather_root: int = -1, d_gather=None):
    """Single-process multi-GPU decode through the C ABI: shard d on CUDA device
    devices[d] into the torch tensor d_outs[d] (plans[d]["out_count"] bytes on that
    device); optional gather of every committed span into d_gather (N bytes on
    devices[gather_root]).  Returns (status, per-device kernel ms)."""
    c = _u8(container)
    n = len(devices)
    devs = (ctypes.c_int * n)(*devices)
    outs = (ctypes.c_void_p * n)(*[o.data_ptr() if o is not None else None for o in d_outs])
    ms = (ctypes.c_float * n)()
    rc = load().recoil_multi_decode(c.ctypes.data, c.size, n, devs, outs, gather_root,
                                    d_gather.data_ptr() if d_gather is not None else None, ms)
    if rc in (RECOIL_E_ARG, RECOIL_E_CUDA, RECOIL_E_NOMEM) or rc <= RECOIL_E_BAD_MAGIC and rc >= RECOIL_E_TRUNCATED:
        raise RecoilError(rc, "recoil_multi_decode")
    return rc, list(ms)


def shard_spans(container, world: int) -> list[tuple[int, int, int, int]]:
    """(task_begin, task_end, out_lo, out_hi) of every rank's shard of `container`
    (recoil_shard_plan + the decoder plans; host only, identical on every rank)."""
    c = _u8(container)
    bounds = recoil_shard_plan(c, world)
    spans = []
    for a, b in zip(bounds, bounds[1:]):
        h = recoil_decoder_create(c, a, b)
        p = recoil_decoder_plan(h)
        recoil_decoder_destroy(h)
        spans.append((a, b, p["out_lo"], p["out_hi"]))
    return spans


def gather_spans(span, spans, root: int = 0, out=None, group=None):
    """Optional final gather (north_star: "NCCL is used only for an optional final
    gather"): every rank sends its committed span (a tensor of out_hi - out_lo
    symbols, on its GPU for NCCL) to `root`, which receives them into `out` (a
    tensor of N symbols, allocated if None) with one batch of point-to-point
    operations.  The decode itself has no data-path exchange; this is
    outside the timed decode.  Returns `out` on root, None elsewhere."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    if rank != root:
        dist.batch_isend_irecv([dist.P2POp(dist.isend, span.contiguous(), root, group)])[0].wait()
        return None
    n_total = spans[-1][3]
    if out is None:
        out = torch.empty(n_total, dtype=span.dtype, device=span.device)
    lo, hi = spans[root][2], spans[root][3]
    out[lo:hi].copy_(span)
    ops = [dist.P2POp(dist.irecv, out[spans[r][2]:spans[r][3]], r, group) for r in range(world) if r != root]
    for w in dist.batch_isend_irecv(ops) if ops else []:
        w.wait()
    return out
