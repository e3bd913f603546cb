"""One adaptive decode (latent workload, 2^25 symbols, one split per resident warp) for ncu:
ncu --set full -k regex:recoil_decode_kernel -s 2 -c 1 python tools/profile_adaptive.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2306_12141_b200 import recoil as R
N = 1 << 25
sym, mid, h = synth.latent_workload(N, synth.seed_for(6))
f = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
K = len(h["len"])
warps, sms = R.recoil_decode_occupancy_adaptive(0, K, int(f.size))
c = R.recoil_encode_adaptive(sym, mid, {"base": h["base"], "len": h["len"], "f": f}, 16, warps * sms)
dec = R.GpuDecoder(c, 0)
dec.set_model_ids(mid)
dec.upload()
for _ in range(3):
    dec.decode()
torch.cuda.synchronize()
print("ok", dec.status(), bool((dec.output().cpu().numpy().view(np.uint16) == sym).all()))
