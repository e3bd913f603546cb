"""Longest-task-first plans (recoil_decoder_create_grouped) on finer containers vs the plain
one-wave container: config 2 stream (100 MiB text); L2 flushed before every timed decode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2306_12141_b200 import recoil as R
kind = sys.argv[1] if len(sys.argv) > 1 else "text"
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 100
warps, sms = R.recoil_decode_occupancy(0, 11)
W1 = warps * sms
sym = synth.text_bytes(mib << 20, synth.seed_for(2)) if kind == "text" else synth.exp_bytes(mib << 20, 50, synth.seed_for(3, 50))
f = R.recoil_build_model(synth.histogram(sym), 11)
scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(dec):
    dec.decode(); torch.cuda.synchronize()
    ok = dec.status()[0] == 0 and bool((dec.output().cpu().numpy() == sym).all())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(20):
        scratch.fill_(i & 7)
        e0.record(); dec.decode(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return ok, float(np.median(ts))


plans = {1: [None], 1.5: [None], 2: [None], 3: [None, ([W1], [2])], 4: [None, ([W1], [3]), ([W1], [2])],
         6: [([W1], [4]), ([W1], [3])], 8: [([W1], [6]), ([W1], [5]), ([W1], [4])]}
for wv, ps in plans.items():
    c = R.recoil_encode(sym, f, 11, int(W1 * wv))
    for g in ps:
        dec = R.GpuDecoder(c, 0, grouped=(g[0] + [1 << 30], g[1] + [1]) if g else None)
        dec.upload()
        ok, ms = timed(dec)
        nt = dec.plan["n_tasks"]
        dec.close()
        print(f"{kind}{mib} container {wv} waves ({R.recoil_inspect(c)['n_splits']} splits) plan={g} tasks={nt} ok={ok} "
              f"ms={ms:.4f} GB/s={len(sym)/ms/1e6:.1f}", flush=True)
