#!/usr/bin/env python3
"""Benchmark: Recoil parallel rANS decode on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config config2] [--impl reference]

A *step* is one pass of the whole hot path over one synthetic
stream: the sm_100a decode kernel over every split task of this rank's shard
(task table, LUT and word slice already resident in HBM; row a1, the
host-side task-table expansion, is part of the e2e leg).  ``value`` is the
whole-job decoded GB/s = symbols decoded by all ranks per step x K / max over
ranks of the device time of the K steps (CUDA events on the decode stream,
L2 flushed with a 256 MiB write before every step, outside the events).

Multi-GPU (torchrun, one process per GPU): one stream of N x the config's
size is sharded by contiguous split ranges (recoil_shard_plan), each rank
decodes its own shard; no collective on the data path -> "scaling": "weak".

``--impl reference`` times the oracle (plain C, single thread) -- this tier's
reference arm -- on a bounded sample of the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "decoded GB/s per GPU and 8×B200 box; compressed-size overhead vs split count"

CONFIGS = {
    # name: (kind, symbols, lambda, description)  -- BASELINE.json "configs"
    "config1": ("exp", 1 << 20, 50.0, "1 MiB exponential (lambda=50) bytes, n=11, 16 splits"),
    "config2": ("text", 100 << 20, 0.0, "100 MiB text-like (Zipf-96, ~5.09 bit/B) bytes, n=11, "
                                         "splits tuned to the kernel's resident warps"),
    "config3": ("exp", 1 << 30, 50.0, "1 GiB exponential (lambda=50) bytes, n=11, occupancy-tuned splits"),
    "config4": ("exp", 1 << 30, 50.0, "1 GiB exponential (lambda=50) bytes, n=11, one encode with 65536 splits "
                                      "combined (P:266-272) to --combine-to splits"),
    "config5": ("image", 1 << 30, 0.0, "image-residual-like bytes (Laplace mixture, ~2.3 bit/B), n=11, "
                                       "sharded by split range (1 GiB per GPU)"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


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


def make_stream(cfg: str, world: int, lam_override: float = 0.0):
    import synth
    kind, n, lam, _ = CONFIGS[cfg]
    lam = lam_override or lam
    n_total = n * world
    sym = synth.workload(kind, n_total, seed=synth.seed_for(int(cfg[-1]), lam), lam=lam or 50.0)
    return sym


def synth_histogram(sym):
    import synth
    return synth.histogram(sym)  # chunked: no 8-byte-per-symbol temporary at the 8 GiB config


def cpu_oracle_decode_rate(container: np.ndarray, sample_tasks: int | None, reps: int = 1):
    """Time the oracle (plain C, single thread) decoding `sample_tasks` evenly spaced tasks
    (None = every task).  Returns (GB/s, symbols per rep, seconds per rep, description)."""
    import oracle
    c = container.tobytes()
    info = oracle.container_info(c)
    M, N = info["M"], info["N"]
    out = np.zeros(max(N, 1), dtype=np.uint8)
    if sample_tasks is None or sample_tasks >= M:
        best = None
        for _ in range(reps):
            t0 = time.perf_counter()
            out = oracle.recoil_decode(c)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return N / best / 1e9, N, best, f"oracle or_recoil_decode of all {M} tasks ({N} symbols), best of {reps}"
    tasks = np.unique(np.linspace(0, M - 1, sample_tasks).astype(int))
    best, nsym = None, 0
    for _ in range(reps):
        t0 = time.perf_counter()
        _, nsym = oracle.recoil_decode_tasks(c, tasks, out)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return nsym / best / 1e9, nsym, best, f"oracle or_recoil_decode_tasks on {len(tasks)} of {M} tasks ({nsym} symbols)"


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


def peak_hbm() -> float:
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs") or 6650.0)
    except Exception:
        return 6650.0


def adaptive_extra(args, local, stream, timed_decode, peak):
    """NEXT rows 1 + 4: the adaptive codec (index-keyed Gaussian models, 16-bit symbols, n = 16) on the
    latent workload, 2^25 symbols, one split per resident warp."""
    import synth
    from paper_2306_12141_b200 import recoil as R
    N = 1 << 25
    sym, mid, h = synth.latent_workload(N, synth.seed_for(6))
    f = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
    models = {"base": h["base"], "len": h["len"], "f": f}
    K = len(h["len"])
    warps, sms = R.recoil_decode_occupancy_adaptive(local, K, int(f.size))
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
    dec.close()
    return {"value": round(2 * N / (ms / 1e3) / 1e9, 2), "unit": "GB/s (16-bit symbols written)",
            "symbols_per_s": round(N / (ms / 1e3), 1), "ms_per_step": round(ms, 4), "bit_exact": ok,
            "n_symbols": N, "splits": info["n_splits"], "models": len(h["len"]), "prob_bits": 16,
            "bits_per_symbol": round(8 * len(c) / N, 3), "resident_warps_per_sm": warps,
            "roofline": {"bound": "hbm", "achieved": round(alg / (ms / 1e3) / 1e9, 1), "peak": peak,
                         "frac": round(alg / (ms / 1e3) / 1e9 / peak, 4)},
            "note": "recoil_decode_adaptive: per symbol a model id (u8) keys one of 64 discretised Gaussians "
                    "(P:227 (3), P:514); coarse bucket + binary search in shared-memory model tables"}


def run_reference(args, rank, world):
    """Reference arm of this tier: the oracle as it stands, on the host cores."""
    if rank != 0:
        return 0
    import oracle  # noqa: F401
    from paper_2306_12141_b200 import recoil as R
    sym = make_stream(args.config, world, args.lam)
    f = R.recoil_build_model(synth_histogram(sym), 11)
    # same split count as our arm: waves x 48 resident warps/SM (the decode kernel's occupancy at n = 11)
    # x SMs per GPU; the SM count is read from torch, not from our library
    import torch
    sms = torch.cuda.get_device_properties(0).multi_processor_count if torch.cuda.is_available() else 148
    waves = args.waves or (1 if args.config == "config2" else 1.5)
    M = args.splits or (16 if args.config == "config1" else int(round(48 * sms * waves))) * world
    c = R.recoil_encode(sym, f, 11, M)
    M = R.recoil_inspect(c)["n_splits"]
    per_step = max(1, M // 64)  # ~1/64 of the stream per step: bounded sample
    times, nsyms = [], []
    for i in range(args.warmup + args.steps):
        gbs, nsym, dt, desc = cpu_oracle_decode_rate(c, per_step)
        if i >= args.warmup:
            times.append(dt)
            nsyms.append(nsym)
    total_t, total_n = sum(times), sum(nsyms)
    value = total_n / total_t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * total_t / len(times), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": args.config + ": " + CONFIGS[args.config][3], "n_symbols": int(len(sym)),
                   "splits": M, "prob_bits": 11, "lanes": 32},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"{per_step} evenly spaced split tasks per step ({desc.split('(')[-1][:-1]})"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="config2", choices=sorted(CONFIGS))
    ap.add_argument("--no-adaptive", action="store_true", help="skip the adaptive-codec extra")
    ap.add_argument("--gather", action="store_true",
                    help="N > 1: time the optional NCCL gather of the ranks' spans to rank 0 (outside the decode)")
    ap.add_argument("--waves", type=float, default=0,
                    help="splits per GPU = waves x resident warps; 0 = per-config default: configs 3/5 1.5 (the "
                         "kernel runs 2 CTAs per SM and the SM schedulers favour the first, whose warps then take the "
                         "last half wave; DESIGN.md §13), config 2 1 (one split per resident warp: equal GB/s, and "
                         "the closest to the partitioned baseline at the same count)")
    ap.add_argument("--splits", type=int, default=0, help="override the split count per GPU")
    ap.add_argument("--combine-to", type=int, default=2048, help="config4: target split count")
    ap.add_argument("--chunks", type=int, default=8, help="e2e pipeline chunks per GPU")
    ap.add_argument("--streams", type=int, default=3, help="e2e pipeline streams per GPU")
    ap.add_argument("--lam", type=float, default=0.0, help="config3/4: override lambda")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-extra", action="store_true", help="skip partitioned / size-overhead legs")
    args = ap.parse_args()
    rank, world, local = dist_env()
    if args.gpus != world and world > 1:
        log(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}")
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    from paper_2306_12141_b200 import recoil as R
    import __graft_entry__
    if rank == 0 or not os.path.exists(R.LIB_PATH):
        __graft_entry__.build()
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        # control plane only (barriers, max-over-ranks timing): the decode has no
        # data-path exchange, so no NCCL collective is on the timed path
        import torch.distributed as dist
        dist.init_process_group("gloo")
        pg = dist
        dist.barrier()
    R.load()

    # ---------------- setup (untimed): synthetic stream, encode, shard plan ----------------
    t_setup = time.perf_counter()
    sym = make_stream(args.config, world, args.lam)
    N_total = len(sym)
    hist = synth_histogram(sym)
    f = R.recoil_build_model(hist, 11)
    warps, sms = R.recoil_decode_occupancy(local, 11)
    if not args.waves:
        args.waves = 1 if args.config == "config2" else 1.5
    M_gpu = args.splits or (16 if args.config == "config1" else int(round(warps * sms * args.waves)))
    if args.config == "config4":
        c_full = R.recoil_encode(sym, f, 11, 65536 * world)
        M_gpu = args.combine_to
        c = R.recoil_combine_splits(c_full, M_gpu * world)
        del c_full
    else:
        c = R.recoil_encode(sym, f, 11, M_gpu * world)
    info = R.recoil_inspect(c)
    M = info["n_splits"]
    bounds = R.recoil_shard_plan(c, world)
    a, b = bounds[rank], bounds[rank + 1]
    pinned = torch.empty(len(c), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = c
    cont = pinned.numpy()
    stream = torch.cuda.Stream(dev)
    dec = R.GpuDecoder(cont, local, a, b, stream=stream)
    plan = dec.plan
    dec.upload()
    torch.cuda.synchronize(dev)
    setup_s = time.perf_counter() - t_setup
    n_rank = plan["out_hi"] - plan["out_lo"]
    words_rank = plan["word_count"]
    alg_bytes = n_rank + 2 * min(words_rank, max(0, info["n_words"] - plan["word_lo"])) + plan["workspace_bytes"]
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    # correctness of this rank's span before timing (bit-exact vs the input = the decode's definition)
    dec.decode()
    rc, bad = dec.status()
    got = dec.output().cpu().numpy()
    ok = rc == 0 and bool((got == sym[plan["out_lo"]:plan["out_hi"]]).all())
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
    # recoil_pipeline_*: per step the host parses the container and expands the
    # task table (a1) chunk by chunk, H2D of tables + word slices from pinned memory,
    # the kernels, D2H of the symbols into pinned memory, status read; chunks on 3
    # streams so copies overlap kernels and each other.
    out_host = torch.empty(max(N_total, 16), dtype=torch.uint8, pin_memory=True)
    pipe = R.HostPipeline(cont, local, n_chunks=args.chunks, n_streams=args.streams, task_begin=a, task_end=b)
    e2e_times = []
    steps_e2e = max(3, min(args.steps, 20))
    for i in range(args.warmup + steps_e2e):
        torch.cuda.synchronize(dev)
        if pg:
            pg.barrier()
        t0 = time.perf_counter()
        pipe.run(out_host)
        rc_e2e, _ = pipe.status()
        dt = time.perf_counter() - t0
        if rc_e2e != 0:
            ok = False
        if i >= args.warmup:
            e2e_times.append(dt)
    e2e_launches = pipe.launches()
    pipe.close()
    e2e_s = float(np.mean(e2e_times))
    if pg:
        t = torch.tensor([e2e_s], dtype=torch.float64)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = N_total / e2e_s / 1e9
    ok = ok and bool((out_host.numpy()[plan["out_lo"]:plan["out_hi"]] == sym[plan["out_lo"]:plan["out_hi"]]).all())

    extra = {}
    if pg and args.gather:
        # row a10: optional final gather of every rank's committed span to rank 0 over NCCL
        # (its own process group; the timed decode above has no data-path exchange)
        nccl = pg.new_group(backend="nccl")
        spans = R.shard_spans(cont, world)
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
        gok = bool((full.cpu().numpy() == sym).all()) if rank == 0 else True
        extra["gather"] = {"ms": round(float(t.item()) * 1e3, 3), "bytes": int(N_total - n_rank) if rank == 0 else 0,
                           "GB/s_into_root": round((N_total - n_rank) / float(t.item()) / 1e9, 2), "bit_exact": gok,
                           "backend": "nccl", "note": "rank spans -> rank 0, batched point-to-point; not in value"}
    if rank == 0 and not args.no_extra:
        # the paper's comparison: conventional partitioned decoder at the same count
        pc = R.recoil_partitioned_encode(sym, f, 11, M)
        pbounds = R.recoil_shard_plan(pc, world)
        pdec = R.GpuDecoder(pc, local, pbounds[0], pbounds[1], stream=stream)
        pdec.upload()
        pt = timed_decode(pdec, args.steps, args.warmup) if world == 1 else None
        pn = pdec.plan["out_hi"] - pdec.plan["out_lo"]
        pdec.decode()
        pok = pdec.status()[0] == 0 and bool((pdec.output().cpu().numpy() ==
                                              sym[pdec.plan["out_lo"]:pdec.plan["out_hi"]]).all())
        if pt:
            extra["partitioned_baseline"] = {
                "value": round(pn * args.steps / (sum(pt) / 1e3) / 1e9, 2), "unit": "GB/s",
                "ms_per_step": round(float(np.mean(pt)), 4), "partitions": M, "bit_exact": pok,
                "container_bytes": int(len(pc))}
        c1 = R.recoil_encode(sym, f, 11, 1)
        p1 = R.recoil_partitioned_encode(sym, f, 11, 1)
        small = R.recoil_combine_splits(c, 16)
        extra["size_overhead"] = {
            "baseline_bytes_M1": int(len(c1)),
            "recoil": {"splits": M, "bytes": int(len(c)), "overhead_bytes": int(len(c) - len(c1)),
                       "bytes_per_split": round((len(c) - len(c1)) / max(1, M - 1), 2)},
            "partitioned": {"partitions": M, "bytes": int(len(pc)), "overhead_bytes": int(len(pc) - len(p1)),
                            "bytes_per_partition": round((len(pc) - len(p1)) / max(1, M - 1), 2)},
            "recoil_combined_to_16": {"bytes": int(len(small)), "overhead_bytes": int(len(small) - len(c1))},
        }
        pdec.close()
        if world == 1 and args.config == "config2" and not args.splits:
            # Z26: BASELINE's "~20k-warp occupancy" split count (3 waves of resident warps)
            M20 = 3 * warps * sms
            c20 = R.recoil_encode(sym, f, 11, M20)
            d20 = R.GpuDecoder(c20, local, stream=stream)
            d20.upload()
            d20.decode()
            ok20 = d20.status()[0] == 0 and bool((d20.output().cpu().numpy() == sym).all())
            t20 = timed_decode(d20, args.steps, args.warmup)
            d20.close()
            p20 = R.recoil_partitioned_encode(sym, f, 11, M20)  # the partitioned baseline at the same count
            q20 = R.GpuDecoder(p20, local, stream=stream)
            q20.upload()
            q20.decode()
            pok20 = q20.status()[0] == 0 and bool((q20.output().cpu().numpy() == sym).all())
            tp20 = timed_decode(q20, args.steps, args.warmup)
            q20.close()
            extra["config2_20k"] = {"value": round(N_total * args.steps / (sum(t20) / 1e3) / 1e9, 2), "unit": "GB/s",
                                    "splits": R.recoil_inspect(c20)["n_splits"], "bit_exact": ok20,
                                    "ms_per_step": round(float(np.mean(t20)), 4),
                                    "partitioned_baseline": {
                                        "value": round(N_total * args.steps / (sum(tp20) / 1e3) / 1e9, 2),
                                        "unit": "GB/s", "partitions": M20, "bit_exact": pok20}}
        if world == 1 and not args.no_adaptive:
            extra["adaptive_latent"] = adaptive_extra(args, local, stream, timed_decode, peak_hbm())
    cpu = None
    if rank == 0 and not args.no_cpu:
        gbs, nsym, dt, desc = cpu_oracle_decode_rate(c, None if N_total <= (256 << 20) else 256, reps=1)
        cpu = {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": desc, "seconds": round(dt, 3)}
        t0 = time.perf_counter()
        threads = os.cpu_count() or 1
        out_cpu = R.recoil_decode_cpu_ex(cont, threads, R.RECOIL_CPU_SCALAR)
        dt_mt = time.perf_counter() - t0
        extra["cpu_mt_library"] = {"value": round(N_total / dt_mt / 1e9, 4), "unit": "GB/s", "threads": threads,
                                   "bit_exact": bool((out_cpu == sym).all()),
                                   "note": "recoil_decode_cpu_ex(SCALAR): scalar MT host decoder (baseline, not a fallback)"}
        if R.recoil_cpu_simd():
            t0 = time.perf_counter()
            out_cpu = R.recoil_decode_cpu_ex(cont, threads, 0)
            dt_mt = time.perf_counter() - t0
            extra["cpu_mt_avx512"] = {"value": round(N_total / dt_mt / 1e9, 4), "unit": "GB/s", "threads": threads,
                                      "bit_exact": bool((out_cpu == sym).all()),
                                      "note": "recoil_decode_cpu: AVX-512 MT host decoder (NEXT row 3; baseline)"}

    prof = {}
    pf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(pf):
        try:
            prof = json.load(open(pf)).get(f"{args.config}:{M_gpu}", {})
        except Exception:
            prof = {}
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = peaks.get("hbm_gbs") or 6650.0
    traffic = prof.get("dram_bytes_per_launch")

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": args.config + ": " + CONFIGS[args.config][3], "n_symbols": int(N_total),
                       "n_symbols_per_gpu": int(CONFIGS[args.config][1]), "splits": int(M),
                       "splits_rule": (f"65536 x {world} encoded, combined to {M_gpu} x {world}"
                                       if args.config == "config4" else
                                       f"{args.waves} waves x {warps} resident warps/SM x {sms} SMs per GPU"
                                       if not args.splits and args.config != "config1" else "fixed"),
                       "lambda": (args.lam or CONFIGS[args.config][2]) if CONFIGS[args.config][0] == "exp" else None,
                       "compressed_bytes": int(len(c)), "prob_bits": 11, "lanes": 32,
                       "parallelism": f"split-range shards x{world}",
                       "l2": "flushed before every timed step (256 MiB write, outside the events)"},
            "bit_exact": ok,
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic,
                         "kernel": "recoil_decode_kernel<11>",
                         "algorithmic_bytes_per_launch": int(alg_bytes),
                         "note": "achieved = (decoded bytes written + compressed words read + task table) / "
                                 "event-timed decode; peak = MEASURED_PEAKS.json hbm_gbs (burst)"},
            "roofline_smem": smem_roofline(prof, my_avg_ms, clocks, sms),
            "cpu_baseline": cpu,
            "e2e": {"value": round(e2e_value, 3), "unit": "GB/s",
                    "h2d_bytes_per_step": int(plan["upload_bytes"]), "d2h_bytes_per_step": int(n_rank),
                    "chunks": args.chunks, "streams": args.streams, "kernel_launches_per_step": int(e2e_launches),
                    "note": "recoil_pipeline_run + status per step: host parse + task expansion (a1) per chunk, "
                            "H2D tables + words from pinned memory, kernels, D2H of the symbols to pinned "
                            "memory, 3 streams overlapping; wall clock, max over ranks"},
            "gpu_launches": int(args.steps * dec.launches()),
            "clocks": clocks.report(),
            "setup_s": round(setup_s, 2),
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
