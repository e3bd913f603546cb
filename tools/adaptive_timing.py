"""Adaptive decode timing (latent, 2^25 symbols, one split per resident warp), CUDA events."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2306_12141_b200 import recoil as R
N = int(os.environ.get("AD_N", 1 << 25))
sym, mid, h = synth.latent_workload(N, synth.seed_for(6))
f = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
K = len(h["len"])
warps, sms = R.recoil_decode_occupancy_adaptive(0, K, int(f.size))
WAVES = float(os.environ.get("AD_WAVES", 1))
c = R.recoil_encode_adaptive(sym, mid, {"base": h["base"], "len": h["len"], "f": f}, 16, int(warps * sms * WAVES))
dec = R.GpuDecoder(c, 0)
dec.set_model_ids(mid)
dec.upload()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for i in range(25):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dec.decode(); e1.record(); torch.cuda.synchronize()
    if i >= 5: ts.append(e0.elapsed_time(e1))
ok = dec.status()[0] == 0 and bool((dec.output().cpu().numpy().view(np.uint16) == sym).all())
ms = float(np.median(ts))
print(os.environ.get("RECOIL_LIB", "default"), f"N {N} waves {WAVES} warps/SM {warps} ms {ms:.4f} Gsym/s {N/ms/1e6:.1f} ok {ok}")
