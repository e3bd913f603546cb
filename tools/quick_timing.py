import time, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2306_12141_b200 import recoil as R
warps, sms = R.recoil_decode_occupancy(0, 11)
print("occupancy warps/SM", warps, "SMs", sms)
sym = synth.text_bytes(100 << 20, synth.seed_for(2))
f = R.recoil_build_model(synth.histogram(sym), 11)
waves = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4,6,8").split(",")]
for kind in ("recoil", "part"):
    for wv in waves:
        M = warps * sms * wv
        c = R.recoil_encode(sym, f, 11, M) if kind == "recoil" else R.recoil_partitioned_encode(sym, f, 11, M)
        dec = R.GpuDecoder(c, 0); dec.upload(); dec.decode(); torch.cuda.synchronize()
        st = dec.status(); ok = (dec.output().cpu().numpy() == sym).all()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(20):
            e0.record(); dec.decode(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(f"{kind:6s} waves={wv} M={M} status={st} ok={ok} ms={ms:.4f} GB/s={len(sym)/ms/1e6:.1f} ratio={len(c)/len(sym):.4f}", flush=True)
        dec.close()
