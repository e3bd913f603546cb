#!/usr/bin/env python3
"""Benchmark: Recoil parallel rANS decode on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config config5] [--impl reference]

A *step* is one pass of the whole hot path over one synthetic
stream: the sm_100a decode kernel over every split task of this rank's shard
(task table, LUT and word slice already resident in HBM; row a1, the host-side
part of the task-table expansion, is part of the e2e leg).  ``value`` is the
whole-job decoded GB/s = symbols decoded by all ranks per step x K / max over
ranks of the device time of the K steps (CUDA events on the decode stream, L2
flushed with a 256 MiB write before every step, outside the events).

Default workload: BASELINE config 5, ONE 8 GiB image-residual-like stream,
encoded once (serial) with the split count of 8 GPUs (8 x 1.5 waves of the
kernel's resident warps).  N GPUs decode it by split range (§8(e)) with no
data-path collective; a decoder with fewer GPUs first shrinks the split metadata
to its own parallelism with recoil_combine_splits ("decoder-adaptive
scalability", one encode for every client), so every GPU runs 1.5 waves of tasks.
The total work is fixed -> "scaling": "strong".  Configs 1-4 are weak-scaled
(N x the per-GPU size).

Multi-rank setup: rank 0 synthesises and encodes once and shares the container
through a file; every rank regenerates only its own output span for the
bit-exact check (counter-based generator), pins only its word slice and its
output span.

``--impl reference`` times this tier's reference arm -- the oracle (plain C,
single thread) -- on a bounded sample of the same workload (rank 0 only): the
leading slice of the same seeded stream, encoded BY THE ORACLE at the same
symbols per split, parsed once outside the timed loop.  No librecoil code runs
in that arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "decoded GB/s per GPU and 8×B200 box; compressed-size overhead vs split count"
GIB = 1 << 30

CONFIGS = {
    # name: (kind, symbols, lambda, strong, description) -- BASELINE.json "configs"
    "config1": ("exp", 1 << 20, 50.0, False, "1 MiB exponential (lambda={lam:g}) bytes per GPU, n=11, 16 splits"),
    "config2": ("text", 100 << 20, 0.0, False, "100 MiB text-like (Zipf-96, ~5.09 bit/B) bytes per GPU, n=11, "
                                               "splits tuned to the kernel's resident warps"),
    "config3": ("exp", GIB, 50.0, False, "1 GiB exponential (lambda={lam:g}) bytes per GPU, n=11, "
                                         "occupancy-tuned splits"),
    "config4": ("exp", GIB, 50.0, False, "1 GiB exponential (lambda={lam:g}) bytes per GPU, n=11, one encode with "
                                         "65536 splits combined (P:266-272) to --combine-to splits"),
    "config5": ("image", 8 * GIB, 0.0, True, "one 8 GiB image-residual-like stream (Laplace mixture, ~2.3 bit/B), "
                                             "n=11, encoded with 8 GPUs' splits, combined to each decoder's "
                                             "parallelism, sharded by split range over the GPUs"),
}
STRONG_ENCODE_GPUS = 8  # config 5 is encoded once for an 8-GPU box (BASELINE config 5)
WAVES = 1.5             # splits per GPU = 1.5 x resident warps (Z26 / §13)
KERNEL_WARPS_PER_SM = 48  # the n = 11 kernel's resident warps (2 CTAs x 24)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def workload_label(cfg: str, lam: float) -> str:
    return cfg + ": " + CONFIGS[cfg][4].format(lam=lam)


def host_cpu():
    """CPU model, physical cores and logical CPUs of this host."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        import psutil
        phys = psutil.cpu_count(logical=False) or os.cpu_count() or 1
    except Exception:
        phys = os.cpu_count() or 1
    try:
        avail = len(os.sched_getaffinity(0))
    except Exception:
        avail = os.cpu_count() or 1
    return {"model": model, "physical_cores": int(phys), "logical_cpus": int(os.cpu_count() or 1),
            "available_cpus": int(avail)}


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, device_index: int, period_s: float = 0.002):
        self.ok = False
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # no NVML: report that instead of clocks
            self.err = str(e)
        self.period = period_s
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(self.period)

    def sample(self):
        if not self.ok:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            for name, bit in self.REASONS.items():
                if r & bit and name != "gpu_idle":
                    self.reasons.add(name)
        except Exception:
            pass

    def __enter__(self):
        self.sample()
        self._stop.clear()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join()
        self.sample()

    def report(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable: " + self.err}
        return {"sm_mhz": float(statistics.median(self.samples)) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def stream_params(cfg: str, lam_override: float):
    kind, n, lam, strong, _ = CONFIGS[cfg]
    lam = lam_override or lam
    return kind, n, (lam or 50.0), strong


def make_stream(cfg: str, n_total: int, lam_override: float = 0.0, start: int = 0, count: int | None = None):
    """Symbols [start, start + count) of the config's seeded stream of n_total symbols."""
    import synth
    kind, _, lam, _ = stream_params(cfg, lam_override)
    count = n_total - start if count is None else count
    return synth.workload(kind, count, seed=synth.seed_for(int(cfg[-1]), lam if kind == "exp" else 0), lam=lam,
                          start=start)


# warp-instructions per 32-symbol group in the n = 11 kernel's unrolled steady state
# (cuobjdump -sass)
STEADY_INSTR_PER_GROUP = 19


def issue_roofline(prof: dict, avg_ms: float, clocks, sms: int, groups: int):
    """The other binding resource: warp-instruction issue (plain integer ALU path, no tensor cores).
    Peak = 4 schedulers x 1 warp-instruction per cycle per SM x SMs x the SM clock sampled during the run
    (B200_PROFILING.md unit counts).  'achieved' counts the algorithmic instructions: the steady-state
    STEADY_INSTR_PER_GROUP warp-instructions per 32-symbol group (SASS of the unrolled block) x the launch's
    groups; 'measured' is ncu's smsp__inst_executed of the same launch (all overheads included)."""
    if avg_ms <= 0:
        return None
    mhz = (clocks.report() or {}).get("sm_mhz") or 1965.0
    peak = 4 * sms * mhz * 1e6
    alg = STEADY_INSTR_PER_GROUP * groups / (avg_ms / 1e3)
    out = {"bound": "alu", "achieved": round(alg / 1e9, 1), "peak": round(peak / 1e9, 1),
           "unit": "G warp-instructions/s", "frac": round(alg / peak, 4),
           "instructions_per_group": STEADY_INSTR_PER_GROUP}
    inst = prof.get("warp_instructions_per_launch")
    if inst:
        out["measured"] = round(inst / (avg_ms / 1e3) / 1e9, 1)
        out["measured_frac"] = round(inst / (avg_ms / 1e3) / peak, 4)
        out["measured_instructions_per_group"] = round(inst / max(1, groups), 2)
    return out


def peak_hbm() -> float:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs") or 6650.0)
    except Exception:
        return 6650.0


def smem_roofline(prof: dict, avg_ms: float, clocks, sms: int):
    """The kernel's binding resource: shared-memory wavefronts (LUT gather, ring word, staging store;
    DESIGN.md §7) per launch from the ncu capture of the same command (profiles/ncu_traffic.json), over
    the event-timed launch, against 1 wavefront per SM-cycle at the clock sampled during the run."""
    wf = prof.get("smem_wavefronts_per_launch")
    if not wf or avg_ms <= 0:
        return None
    mhz = (clocks.report() or {}).get("sm_mhz") or 1965.0
    peak = sms * mhz * 1e6
    achieved = wf / (avg_ms / 1e3)
    return {"bound": "smem", "achieved": round(achieved / 1e9, 2), "peak": round(peak / 1e9, 2),
            "unit": "G wavefronts/s", "frac": round(achieved / peak, 4), "wavefronts_per_launch": int(wf),
            "source": prof.get("source")}


# ------------------------------------------------------------------------------------------
# reference arm: the oracle, as it stands, on the host cores (rank 0 only); oracle code only
# ------------------------------------------------------------------------------------------

def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import oracle
    import synth
    cfg = args.config
    kind, n_gpu, lam, strong = stream_params(cfg, args.lam)
    n_total = n_gpu if strong else n_gpu * world
    # symbols per split of our arm's decode: 1.5 waves of the kernel's resident warps per GPU
    try:
        import torch
        sms = torch.cuda.get_device_properties(0).multi_processor_count if torch.cuda.is_available() else 148
    except Exception:
        sms = 148
    if cfg == "config1":
        splits_per_gpu = 16
    elif cfg == "config4":
        splits_per_gpu = args.combine_to
    else:
        splits_per_gpu = args.splits or int(round(KERNEL_WARPS_PER_SM * sms * (args.waves or WAVES)))
    sym_per_split = n_gpu / (world if strong else 1) / splits_per_gpu
    # bounded sample: the leading slice of the same stream, encoded by the oracle at that density
    n_sample = int(min(n_total, args.ref_sample_mib << 20))
    m_sample = max(1, int(round(n_sample / sym_per_split)))
    sym = make_stream(cfg, n_total, args.lam, 0, n_sample)
    f = oracle.build_model(synth.histogram(sym), 11)
    t0 = time.perf_counter()
    c = oracle.recoil_encode(sym, f, 11, m_sample)
    enc_s = time.perf_counter() - t0
    opened = oracle.Opened(c)  # parse once, outside the timed loop
    M = opened.info["M"]
    out = np.bitwise_not(sym)  # every byte differs from the input until a task writes it
    per_step = max(1, min(M, args.ref_tasks))
    times, nsyms = [], []
    for i in range(args.warmup + args.steps):
        tasks = [(i * per_step + k) % M for k in range(per_step)]
        t0 = time.perf_counter()
        nsym = opened.decode_tasks(tasks, out)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            nsyms.append(nsym)
    opened.close()
    written = out != np.bitwise_not(sym)
    ok = bool(written.any()) and bool(np.array_equal(out[written], sym[written]))
    total_t, total_n = sum(times), sum(nsyms)
    value = total_n / total_t / 1e9
    cpu = host_cpu()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total_t / len(times), 3),
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": workload_label(cfg, lam), "n_symbols": int(n_total), "prob_bits": 11, "lanes": 32,
                   "symbols_per_split": round(sym_per_split, 1)},
        "bit_exact": ok,
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"leading {n_sample >> 20} MiB of the same stream, encoded by the oracle "
                                   f"(or_recoil_encode, {enc_s:.1f} s, untimed) into {M} splits of "
                                   f"~{sym_per_split / 1e3:.0f}k symbols; per step or_opened_decode_tasks on "
                                   f"{per_step} consecutive tasks (container parsed once, outside the timing)",
                         "cpu": cpu},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------

def adaptive_extra(args, local, stream, timed_decode, peak, log2n: int = 25):
    """NEXT rows 1 + 4: the adaptive codec (index-keyed Gaussian models, 16-bit symbols, n = 16) on the
    latent workload, 2^log2n symbols (2^25: ~15 div2k-sized latents; 2^27
    as well, where the split heuristic's uneven tasks weigh less), one split per
    resident warp."""
    import synth
    from paper_2306_12141_b200 import recoil as R
    N = 1 << log2n
    sym, mid, h = synth.latent_workload(N, synth.seed_for(6))
    f = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
    models = {"base": h["base"], "len": h["len"], "f": f}
    warps, sms = R.recoil_decode_occupancy_adaptive(local, len(h["len"]), int(f.size))
    c = R.recoil_encode_adaptive(sym, mid, models, 16, warps * sms)
    info = R.recoil_inspect(c)
    dec = R.GpuDecoder(c, local, stream=stream)
    dec.set_model_ids(mid)
    dec.upload()
    dec.decode()
    rc, _ = dec.status()
    ok = rc == 0 and bool((dec.output().cpu().numpy().view(np.uint16) == sym).all())
    t = timed_decode(dec, args.steps, args.warmup)
    ms = float(np.mean(t))
    alg = 2 * N + N + 2 * info["n_words"] + dec.plan["workspace_bytes"]  # symbols out + model ids + words
    plan = dec.plan
    dec.close()
    return {"value": round(2 * N / (ms / 1e3) / 1e9, 2), "unit": "GB/s (16-bit symbols written)",
            "symbols_per_s": round(N / (ms / 1e3), 1), "ms_per_step": round(ms, 4), "bit_exact": ok,
            "n_symbols": N, "splits": info["n_splits"], "models": len(h["len"]), "prob_bits": 16,
            "bits_per_symbol": round(8 * len(c) / N, 3), "resident_warps_per_sm": warps,
            "coarse_bits": plan["coarse_bits"], "warps_per_block": plan["warps_per_block"],
            "roofline": {"bound": "hbm", "achieved": round(alg / (ms / 1e3) / 1e9, 1), "peak": peak,
                         "frac": round(alg / (ms / 1e3) / 1e9 / peak, 4)},
            "note": "recoil_decode_adaptive: per symbol a model id (u8) keys one of 64 discretised Gaussians "
                    "(P:227 (3), P:514); coarse bucket + binary search in shared-memory model tables"}


def size_sweep(sym, f, counts):
    """Compressed-size overhead vs split count (BASELINE metric, second half; tab:overhead P:466-512):
    Recoil and the partitioned codec encoded at each count, overhead = size - size at 1."""
    from paper_2306_12141_b200 import recoil as R
    rows = []
    base_r = base_p = None
    for m in counts:
        t0 = time.perf_counter()
        c = R.recoil_encode(sym, f, 11, m)
        enc_s = time.perf_counter() - t0
        p = R.recoil_partitioned_encode(sym, f, 11, m)
        mr = R.recoil_inspect(c)["n_splits"]
        if base_r is None:
            base_r, base_p = len(c), len(p)
        rows.append({"requested": int(m), "recoil_splits": int(mr), "recoil_bytes": int(len(c)),
                     "recoil_overhead_bytes": int(len(c) - base_r),
                     "recoil_bytes_per_split": round((len(c) - base_r) / max(1, mr - 1), 2),
                     "partitioned_bytes": int(len(p)), "partitioned_overhead_bytes": int(len(p) - base_p),
                     "partitioned_bytes_per_partition": round((len(p) - base_p) / max(1, m - 1), 2),
                     "recoil_encode_s": round(enc_s, 2)})
        del c, p
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="config5", choices=sorted(CONFIGS))
    ap.add_argument("--no-adaptive", action="store_true", help="skip the adaptive-codec extra")
    ap.add_argument("--gather", action="store_true",
                    help="N > 1: time the optional NCCL gather of the ranks' spans to rank 0 (outside the decode)")
    ap.add_argument("--waves", type=float, default=0,
                    help=f"splits per GPU = waves x resident warps; 0 = {WAVES} (DESIGN.md §13)")
    ap.add_argument("--splits", type=int, default=0, help="override the split count per GPU")
    ap.add_argument("--combine-to", type=int, default=2048, help="config4: target split count")
    ap.add_argument("--chunks", type=int, default=16, help="e2e pipeline chunks per GPU")
    ap.add_argument("--streams", type=int, default=3, help="e2e pipeline streams per GPU")
    ap.add_argument("--lam", type=float, default=0.0, help="config3/4: override lambda")
    ap.add_argument("--reps", type=int, default=3, help="alternating Recoil / partitioned repetitions (N = 1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample-mib", type=int, default=32, help="reference arm: sample size")
    ap.add_argument("--ref-tasks", type=int, default=4, help="reference arm: tasks decoded per step")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline / host decoder legs")
    ap.add_argument("--no-extra", action="store_true", help="skip partitioned / size-overhead legs")
    ap.add_argument("--size-sweep", action="store_true",
                    help="add the compression-vs-split-count sweep M in {1,16,256,2048,M_occ,65536} (both codecs)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.gpus != world and world > 1:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}")
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    from paper_2306_12141_b200 import recoil as R
    import __graft_entry__
    import synth
    if rank == 0 or not os.path.exists(R.LIB_PATH):
        __graft_entry__.build()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        # control plane only (barriers, max-over-ranks timing, container hand-off): the decode has
        # no data-path exchange, so no collective is on the timed path
        import torch.distributed as dist
        dist.init_process_group("gloo")
        pg = dist
        pg.barrier()
    R.load()
    cfg = args.config
    kind, n_gpu, lam, strong = stream_params(cfg, args.lam)
    N_total = n_gpu if strong else n_gpu * world
    warps, sms = R.recoil_decode_occupancy(local, 11)
    waves = args.waves or WAVES
    per_gpu_splits = (16 if cfg == "config1" else args.combine_to if cfg == "config4" else
                      args.splits or int(round(warps * sms * waves)))

    # ---------------- setup (untimed): rank 0 synthesises and encodes once ----------------
    t_setup = time.perf_counter()
    sym = f_model = None
    share = os.path.join(tempfile.gettempdir(), f"recoil_bench_{os.environ.get('MASTER_PORT', '0')}.bin")
    enc_s = 0.0
    if rank == 0:
        sym = make_stream(cfg, N_total, args.lam)
        f = f_model = R.recoil_build_model(synth.histogram(sym), 11)
        t0 = time.perf_counter()
        if cfg == "config4":
            c_enc = R.recoil_encode(sym, f, 11, 65536 * world)
        elif strong:
            c_enc = R.recoil_encode(sym, f, 11, per_gpu_splits * STRONG_ENCODE_GPUS)
        else:
            c_enc = R.recoil_encode(sym, f, 11, per_gpu_splits * world)
        enc_s = time.perf_counter() - t0
        if world > 1:
            try:
                c_enc.tofile(share)
            except OSError as e:  # no room for a file: hand the container over through the process group
                log(f"container file hand-off failed ({e}); broadcasting over gloo")
                share = None
    if world > 1:
        # the hand-off path (or its failure) is decided by rank 0 and broadcast with the length
        import torch
        meta = torch.tensor([len(c_enc) if rank == 0 else 0, 1 if (rank == 0 and share) else 0], dtype=torch.int64)
        pg.broadcast(meta, 0)
        n_c, by_file = int(meta[0]), bool(meta[1])
        if by_file:
            pg.barrier()
            if rank != 0:
                c_enc = np.fromfile(share, dtype=np.uint8)
            pg.barrier()
            if rank == 0:
                os.unlink(share)
        else:
            buf = torch.from_numpy(c_enc) if rank == 0 else torch.empty(n_c, dtype=torch.uint8)
            step = 256 << 20
            for o in range(0, n_c, step):
                pg.broadcast(buf[o:o + step], 0)
            c_enc = buf.numpy()
    M_enc = R.recoil_inspect(c_enc)["n_splits"]
    # decoder-adaptive scalability: shrink the metadata to this job's parallelism
    target = per_gpu_splits * world
    if target < M_enc:
        t0 = time.perf_counter()
        c = R.recoil_combine_splits(c_enc, target)
        combine_s = time.perf_counter() - t0
    else:
        c, combine_s = c_enc, 0.0
    info = R.recoil_inspect(c)
    M = info["n_splits"]
    bounds = R.recoil_shard_plan(c, world)
    a, b = bounds[rank], bounds[rank + 1]
    stream = torch.cuda.Stream(dev)
    dec = R.GpuDecoder(c, local, a, b, stream=stream)
    plan = dec.plan
    dec.upload()
    torch.cuda.synchronize(dev)
    out_lo, out_hi = plan["out_lo"], plan["out_hi"]
    n_rank = out_hi - out_lo
    want = sym[out_lo:out_hi] if sym is not None else make_stream(cfg, N_total, args.lam, out_lo, n_rank)
    words_rank = plan["word_count"]
    alg_bytes = n_rank + 2 * min(words_rank, max(0, info["n_words"] - plan["word_lo"])) + plan["workspace_bytes"]
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    setup_s = time.perf_counter() - t_setup

    # correctness of this rank's span before timing (bit-exact vs the input = the decode's definition)
    dec.decode()
    rc, bad = dec.status()
    ok = rc == 0 and bool(torch.equal(dec.output(), torch.from_numpy(want).to(dev)))
    if not ok:
        log(f"rank {rank}: decode mismatch rc={rc} bad={bad}")

    def timed_decode(decoder, steps, warmup):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for _ in range(warmup):
            flush_buf.fill_(1)
            decoder.decode()
        torch.cuda.synchronize(dev)
        if pg:
            pg.barrier()
        torch.cuda.synchronize(dev)
        with torch.cuda.stream(stream):
            for i in range(steps):
                flush_buf.fill_(2)      # evict L2 (256 MiB > 126 MB) outside the events
                ev[i][0].record(stream)
                decoder.decode()
                ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        if pg:
            pg.barrier()
        torch.cuda.synchronize(dev)
        return [s.elapsed_time(e) for s, e in ev]

    clocks = ClockSampler(local)
    with clocks:
        times = timed_decode(dec, args.steps, args.warmup)
    total_ms = float(sum(times))
    if pg:
        t = torch.tensor([total_ms], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        total_ms = float(t.item())
        okt = torch.tensor([1 if ok else 0], dtype=torch.int64)
        pg.all_reduce(okt, op=pg.ReduceOp.MIN)
        ok = bool(okt.item())
    value = N_total * args.steps / (total_ms / 1e3) / 1e9
    my_avg_ms = float(np.mean(times))
    achieved = alg_bytes / (my_avg_ms / 1e3) / 1e9

    # ---------------- e2e: host container -> host symbols through the C ABI ----------------
    # recoil_pipeline_*: per step the host parses the container and expands the task table (a1)
    # chunk by chunk, H2D of tables + word slices from pinned memory, the kernels, D2H of the
    # symbols into this rank's pinned span buffer, status read; chunks on 3 streams so copies
    # overlap kernels and each other.  Only the rank's word slice and its span are pinned.
    wbase = len(c) - 2 * info["n_words"]
    pin_lo = (c.ctypes.data + wbase + 2 * plan["word_lo"]) & ~4095
    pin_hi = c.ctypes.data + wbase + 2 * min(info["n_words"], plan["word_lo"] + plan["word_count"])
    cudart = torch.cuda.cudart()
    pinned_ok = pin_hi > pin_lo and int(cudart.cudaHostRegister(pin_lo, pin_hi - pin_lo, 0)) == 0
    out_host = torch.empty(max(n_rank, 16), dtype=torch.uint8, pin_memory=True)
    pipe = R.HostPipeline(c, local, n_chunks=args.chunks, n_streams=args.streams, task_begin=a, task_end=b)
    e2e_times = []
    steps_e2e = max(3, min(args.steps, 10))
    for i in range(min(args.warmup, 3) + steps_e2e):
        torch.cuda.synchronize(dev)
        if pg:
            pg.barrier()
        t0 = time.perf_counter()
        pipe.run(out_host, out_lo)
        rc_e2e, _ = pipe.status()
        dt = time.perf_counter() - t0
        if rc_e2e != 0:
            ok = False
        if i >= min(args.warmup, 3):
            e2e_times.append(dt)
    e2e_launches = pipe.launches()
    pipe.close()
    if pinned_ok:
        cudart.cudaHostUnregister(pin_lo)
    e2e_s = float(np.mean(e2e_times))
    if pg:
        t = torch.tensor([e2e_s], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = N_total / e2e_s / 1e9
    ok = ok and bool(np.array_equal(out_host.numpy()[:n_rank], want))
    del out_host

    extra = {}
    if world == 1:
        # e2e with the on-device metadata path (NEXT 2): per step the host copies the container
        # bytes to the GPU as they are (pinned -> device), the GPU decodes the split metadata and
        # the symbols, and the symbols come back; the host parses only the fixed header
        dd = R.DeviceContainerDecoder(c, local, stream=stream)
        pin_c = torch.empty(len(c), dtype=torch.uint8, pin_memory=True)
        pin_c.numpy()[:] = c
        host_syms = torch.empty(max(N_total, 16), dtype=torch.uint8, pin_memory=True)
        dts = []
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dev_ms = []
        for i in range(min(args.warmup, 3) + steps_e2e):
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            dd.upload(pin_c)
            ev0.record(stream)
            dd.decode()
            ev1.record(stream)
            with torch.cuda.stream(stream):
                host_syms[:N_total].copy_(dd.output(), non_blocking=True)
            drc, _ = dd.status()
            dt = time.perf_counter() - t0
            if i >= min(args.warmup, 3):
                dts.append(dt)
                dev_ms.append(ev0.elapsed_time(ev1))
        dok = drc == 0 and bool(np.array_equal(host_syms.numpy()[:N_total], sym))
        extra["e2e_device_metadata"] = {
            "value": round(N_total / float(np.mean(dts)) / 1e9, 3), "unit": "GB/s", "bit_exact": dok,
            "h2d_bytes_per_step": int(len(c)), "d2h_bytes_per_step": int(N_total),
            "device_parse_and_decode_ms": round(float(np.mean(dev_ms)), 4),
            "device_parse_and_decode_GBs": round(N_total / float(np.mean(dev_ms)) / 1e6, 1),
            "kernel_launches_per_step": int(dd.launches()),
            "note": "recoil_device_upload + recoil_device_decode + D2H: the host reads only the fixed header; "
                    "global series, split-record offsets (speculative chunked parse), LUT and task records are "
                    "built on the GPU; one stream, wall clock"}
        dd.close()
        del pin_c, host_syms
    if pg and args.gather:
        # row a10: optional final gather of every rank's committed span to rank 0 over NCCL
        # (its own process group; the timed decode above has no data-path exchange)
        nccl = pg.new_group(backend="nccl")
        spans = R.shard_spans(c, world)
        full = torch.empty(N_total, dtype=torch.uint8, device=dev) if rank == 0 else None
        gts = []
        for i in range(4):
            torch.cuda.synchronize(dev)
            pg.barrier()
            t0 = time.perf_counter()
            R.gather_spans(dec.output(), spans, root=0, out=full, group=nccl)
            torch.cuda.synchronize(dev)
            gts.append(time.perf_counter() - t0)
        gt = float(np.median(gts[1:]))
        t = torch.tensor([gt], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        gok = bool(torch.equal(full, torch.from_numpy(sym).to(dev))) if rank == 0 else True
        extra["gather"] = {"ms": round(float(t.item()) * 1e3, 3), "bytes": int(N_total - n_rank) if rank == 0 else 0,
                           "GB/s_into_root": round((N_total - n_rank) / float(t.item()) / 1e9, 2), "bit_exact": gok,
                           "backend": "nccl", "note": "rank spans -> rank 0, batched point-to-point; not in value"}
        del full
    if rank == 0 and world == 1 and target < M_enc:
        # the same combine on the GPU (recoil_device_combine, NEXT 2): the encoded container already
        # in device memory shrunk to this job's split count; output byte-identical to the host combine
        d_enc = torch.from_numpy(c_enc).to(dev)
        d_small = R.recoil_device_combine(c_enc, d_enc, target)  # warm-up: the allocator's first blocks
        dts = []
        for i in range(5):
            del d_small  # the next call's output reuses the freed block (no cudaMalloc in the timing)
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            d_small = R.recoil_device_combine(c_enc, d_enc, target)
            dts.append(time.perf_counter() - t0)
        same = bool(d_small.numel() == len(c) and torch.equal(d_small, torch.from_numpy(c).to(dev)))
        extra["device_combine"] = {"ms": round(1e3 * float(np.median(dts)), 3), "host_combine_ms": round(1e3 * combine_s, 3),
                                   "from_splits": int(M_enc), "to_splits": int(M), "byte_identical": same,
                                   "note": "recoil_device_combine wall time (two 8-byte read-backs, the word "
                                           "stream copied device to device) vs recoil_combine_splits on the host"}
        del d_enc, d_small
    if rank == 0 and world == 1 and not args.no_extra:
        # the paper's comparison: conventional partitioned decoder at the same count,
        # alternating with Recoil in one run (median of --reps repetitions of K steps each)
        pc = R.recoil_partitioned_encode(sym, f_model, 11, M)
        pdec = R.GpuDecoder(pc, local, stream=stream)
        pdec.upload()
        pdec.decode()
        pok = pdec.status()[0] == 0 and bool(torch.equal(pdec.output(), torch.from_numpy(sym).to(dev)))
        r_gbs, p_gbs = [], []
        for _ in range(args.reps):
            r_gbs.append(N_total * args.steps / (sum(timed_decode(dec, args.steps, 2)) / 1e3) / 1e9)
            p_gbs.append(N_total * args.steps / (sum(timed_decode(pdec, args.steps, 2)) / 1e3) / 1e9)
        pdec.close()
        extra["partitioned_baseline"] = {
            "value": round(float(np.median(p_gbs)), 2), "unit": "GB/s", "partitions": M, "bit_exact": pok,
            "container_bytes": int(len(pc)), "recoil_median": round(float(np.median(r_gbs)), 2),
            "recoil_over_partitioned": round(float(np.median(r_gbs)) / float(np.median(p_gbs)), 4),
            "reps": args.reps, "recoil_reps": [round(x, 1) for x in r_gbs], "partitioned_reps": [round(x, 1) for x in p_gbs],
            "note": "same split count, same box, alternating K-step repetitions; medians"}
        if M_enc > M:
            # decoder-adaptive scalability: both codecs encoded ONCE with the 8-GPU split
            # count; the Recoil client decodes the same container with fewer splits (its `value`
            # above), a partitioned client must decode every partition of its container
            pce = R.recoil_partitioned_encode(sym, f_model, 11, M_enc)
            qdec = R.GpuDecoder(pce, local, stream=stream)
            qdec.upload()
            qdec.decode()
            qok = qdec.status()[0] == 0 and bool(torch.equal(qdec.output(), torch.from_numpy(sym).to(dev)))
            r2, q2 = [], []
            for _ in range(args.reps):
                r2.append(N_total * args.steps / (sum(timed_decode(dec, args.steps, 2)) / 1e3) / 1e9)
                q2.append(N_total * args.steps / (sum(timed_decode(qdec, args.steps, 2)) / 1e3) / 1e9)
            qdec.close()
            extra["partitioned_same_encode"] = {
                "value": round(float(np.median(q2)), 2), "unit": "GB/s", "partitions": M_enc, "bit_exact": qok,
                "container_bytes": int(len(pce)), "recoil_container_bytes": int(len(c_enc)),
                "recoil_median": round(float(np.median(r2)), 2), "recoil_splits_decoded": M,
                "recoil_over_partitioned": round(float(np.median(r2)) / float(np.median(q2)), 4),
                "reps": args.reps,
                "note": "both codecs encoded once for an 8-GPU box (same split count, Recoil's metadata smaller); "
                        "this one-GPU client: Recoil combines to its parallelism, partitioned decodes every "
                        "partition; alternating repetitions, medians"}
            del pce
        # size overhead at this count; M = 1 containers: Recoil = this container combined to 1 split
        # (= encode at M = 1: same stream, no points), partitioned P = 1 = the same single codec's
        # words + one offset and 32 final states (header + model as the P-partition container)
        c1 = R.recoil_combine_splits(c, 1)
        count = int(np.count_nonzero(f_model))
        p1_len = 28 + 2 + 5 * count + 4 + 4 * 32 + 2 * R.recoil_inspect(c1)["n_words"]
        small = R.recoil_combine_splits(c, 16)
        extra["size_overhead"] = {
            "baseline_bytes_M1": int(len(c1)),
            "recoil": {"splits": M, "bytes": int(len(c)), "overhead_bytes": int(len(c) - len(c1)),
                       "bytes_per_split": round((len(c) - len(c1)) / max(1, M - 1), 2)},
            "partitioned": {"partitions": M, "bytes": int(len(pc)), "overhead_bytes": int(len(pc) - p1_len),
                            "bytes_per_partition": round((len(pc) - p1_len) / max(1, M - 1), 2)},
            "recoil_encoded_splits": {"splits": M_enc, "bytes": int(len(c_enc)),
                                      "overhead_bytes": int(len(c_enc) - len(c1))},
            "recoil_combined_to_16": {"bytes": int(len(small)), "overhead_bytes": int(len(small) - len(c1))},
            "note": "partitioned P = 1 size derived (same single interleaved codec as Recoil M = 1)"}
        del pc, c1, small
        if args.size_sweep:
            extra["size_sweep"] = {"workload": workload_label(cfg, lam),
                                   "rows": size_sweep(sym, f_model, [1, 16, 256, 2048, M, 65536])}
        if cfg == "config2" and not args.splits:
            # Z26: BASELINE's "~20k-warp occupancy" split count (3 waves of resident warps)
            M20 = 3 * warps * sms
            c20 = R.recoil_encode(sym, f_model, 11, M20)
            d20 = R.GpuDecoder(c20, local, stream=stream)
            d20.upload()
            d20.decode()
            ok20 = d20.status()[0] == 0 and bool((d20.output().cpu().numpy() == sym).all())
            p20 = R.recoil_partitioned_encode(sym, f_model, 11, M20)
            q20 = R.GpuDecoder(p20, local, stream=stream)
            q20.upload()
            q20.decode()
            pok20 = q20.status()[0] == 0 and bool((q20.output().cpu().numpy() == sym).all())
            r20, p20g = [], []
            for _ in range(args.reps):
                r20.append(N_total * args.steps / (sum(timed_decode(d20, args.steps, 2)) / 1e3) / 1e9)
                p20g.append(N_total * args.steps / (sum(timed_decode(q20, args.steps, 2)) / 1e3) / 1e9)
            # decoder-side combine of the same 3-wave container to 1.5 waves (in place)
            s20 = R.GpuDecoder(c20, local, stream=stream, subset=M20 // 2)
            s20.upload()
            s20.decode()
            sok20 = s20.status()[0] == 0 and bool((s20.output().cpu().numpy() == sym).all())
            rs20 = [N_total * args.steps / (sum(timed_decode(s20, args.steps, 2)) / 1e3) / 1e9
                    for _ in range(args.reps)]
            s20.close()
            d20.close()
            q20.close()
            extra["config2_20k"] = {"value": round(float(np.median(r20)), 2), "unit": "GB/s",
                                    "decoder_side_combine_to_half": {
                                        "value": round(float(np.median(rs20)), 2), "bit_exact": sok20,
                                        "over_partitioned": round(float(np.median(rs20) / np.median(p20g)), 4),
                                        "note": "the same container decoded with every second split point "
                                                "(recoil_decoder_create_subset)"},
                                    "splits": R.recoil_inspect(c20)["n_splits"], "bit_exact": ok20,
                                    "partitioned_baseline": {"value": round(float(np.median(p20g)), 2),
                                                             "unit": "GB/s", "partitions": M20, "bit_exact": pok20},
                                    "recoil_over_partitioned": round(float(np.median(r20) / np.median(p20g)), 4)}
        if not args.no_adaptive:
            extra["adaptive_latent"] = adaptive_extra(args, local, stream, timed_decode, peak_hbm())
            extra["adaptive_latent_2p27"] = adaptive_extra(args, local, stream, timed_decode, peak_hbm(), 27)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        # the oracle as it stands, one host core, a bounded sample: evenly spaced tasks of this container
        import oracle
        cpuinfo = host_cpu()
        t0 = time.perf_counter()
        opened = oracle.Opened(c)
        open_s = time.perf_counter() - t0
        n_tasks = max(1, min(M, int(round(M * min(1.0, (1 << 30) / N_total)))))
        tasks = np.unique(np.linspace(0, M - 1, n_tasks).astype(np.int64))
        scratch = np.bitwise_not(sym)  # every byte differs from the input until a task writes it
        t0 = time.perf_counter()
        nsym = opened.decode_tasks(tasks, scratch)
        dt = time.perf_counter() - t0
        opened.close()
        cok = int(np.count_nonzero(scratch == sym)) == nsym  # exactly the committed symbols, all correct
        del scratch
        cpu = {"value": round(nsym / dt / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": f"or_opened_decode_tasks on {len(tasks)} evenly spaced of the {M} tasks ({nsym} symbols, "
                         f"{dt:.1f} s); container parsed once ({open_s:.1f} s, untimed)",
               "bit_exact": cok, "cpu": cpuinfo}
        threads = cpuinfo["physical_cores"]  # one thread per physical core, no SMT
        legs = [("cpu_mt_library", R.RECOIL_CPU_SCALAR, "recoil_decode_cpu_ex(SCALAR): scalar MT host decoder")]
        if R.recoil_cpu_simd() >= 1:
            legs.append(("cpu_mt_avx2", R.RECOIL_CPU_AVX2, "recoil_decode_cpu_ex(AVX2): 8 lanes x 4 vectors"))
        if R.recoil_cpu_simd() == 2:
            legs.append(("cpu_mt_avx512", 0, "recoil_decode_cpu: AVX-512, 16 lanes x 2 vectors"))
        for key, flags, note in legs:
            t0 = time.perf_counter()
            out_cpu = R.recoil_decode_cpu_ex(c, threads, flags)
            dt_mt = time.perf_counter() - t0
            extra[key] = {"value": round(N_total / dt_mt / 1e9, 4), "unit": "GB/s", "threads": threads,
                          "bit_exact": bool(np.array_equal(out_cpu, sym)), "cpu": cpuinfo,
                          "note": note + " (NEXT row 3, P:429; a host baseline, not a fallback)"}
            del out_cpu

    prof = {}
    pf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(pf):
        try:
            prof = json.load(open(pf)).get(f"{cfg}:{plan['n_tasks']}", {})
        except Exception:
            prof = {}
    peak = peak_hbm()
    traffic = prof.get("dram_bytes_per_launch")

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": workload_label(cfg, lam), "n_symbols": int(N_total),
                       "n_symbols_per_gpu": int(N_total // world), "splits": int(M),
                       "splits_encoded": int(M_enc),
                       "splits_rule": (f"encoded with 65536 x {world}, combined to {per_gpu_splits} x {world}"
                                       if cfg == "config4" else
                                       f"encoded with {STRONG_ENCODE_GPUS} x {per_gpu_splits} "
                                       f"({waves} waves x {warps} resident warps/SM x {sms} SMs), combined "
                                       f"(recoil_combine_splits, P:266-272) to {per_gpu_splits} x {world}"
                                       if strong else
                                       f"{waves} waves x {warps} resident warps/SM x {sms} SMs per GPU"
                                       if not args.splits and cfg != "config1" else "fixed"),
                       "lambda": lam if kind == "exp" else None,
                       "compressed_bytes": int(len(c)), "prob_bits": 11, "lanes": 32,
                       "parallelism": f"split-range shards x{world}",
                       "l2": "flushed before every timed step (256 MiB write, outside the events)"},
            "bit_exact": ok,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": "recoil_decode_kernel<11>",
                         "algorithmic_bytes_per_launch": int(alg_bytes),
                         "note": "achieved = (decoded bytes written + compressed words read + task table) / "
                                 "event-timed decode (rank 0); peak = MEASURED_PEAKS.json hbm_gbs (burst)"},
            "roofline_smem": smem_roofline(prof, my_avg_ms, clocks, sms),
            "roofline_issue": issue_roofline(prof, my_avg_ms, clocks, sms, (n_rank + 31) // 32),
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": int(plan["upload_bytes"]), "d2h_bytes_per_step": int(n_rank),
                    "chunks": args.chunks, "streams": args.streams, "kernel_launches_per_step": int(e2e_launches),
                    "pinned": "word slice registered in place + span-sized output" if pinned_ok else
                              "output span pinned; container pageable",
                    "note": "recoil_pipeline_run_at + status per step: host parse + task expansion (a1) per chunk, "
                            "H2D tables + words, kernels, D2H of the symbols to pinned memory, 3 streams "
                            "overlapping; wall clock, max over ranks"},
            "gpu_launches": int(args.steps * dec.launches()),
            "clocks": clocks.report(),
            "setup_s": round(setup_s, 2), "encode_s": round(enc_s, 2), "combine_s": round(combine_s, 2),
        }
        line.update(extra)
        print(json.dumps(line), flush=True)
    dec.close()
    if pg:
        pg.barrier()
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
