"""Decode GB/s vs stream size and split waves (fixed-overhead vs per-group cost), L2 not flushed.
usage: python tools/size_sweep.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2306_12141_b200 import recoil as R
warps, sms = R.recoil_decode_occupancy(0, 11)
for kind, mib in (("text", 100), ("text", 200), ("text", 400), ("exp", 100), ("exp", 400)):
    sym = synth.text_bytes(mib << 20, synth.seed_for(2)) if kind == "text" else synth.exp_bytes(mib << 20, 50, synth.seed_for(3, 50))
    f = R.recoil_build_model(synth.histogram(sym), 11)
    for wv in (1, 2, 3):
        M = warps * sms * wv
        c = R.recoil_encode(sym, f, 11, M)
        dec = R.GpuDecoder(c, 0); dec.upload(); dec.decode(); torch.cuda.synchronize()
        ok = dec.status()[0] == 0 and bool((dec.output().cpu().numpy() == sym).all())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(20):
            e0.record(); dec.decode(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(f"{kind:4s} {mib:4d} MiB waves={wv} M={M} ok={ok} ms={ms:.4f} GB/s={len(sym)/ms/1e6:.1f}", flush=True)
        dec.close()
