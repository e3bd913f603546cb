"""Launch the decode kernel a few times on a BASELINE workload (for ncu captures).
usage: python tools/profile_decode.py [config2|config1|exp50_1g] [recoil|part] [reps] [waves]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2306_12141_b200 import recoil as R
cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
kind = sys.argv[2] if len(sys.argv) > 2 else "recoil"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
waves = float(sys.argv[4]) if len(sys.argv) > 4 else 0
warps, sms = R.recoil_decode_occupancy(0, 11)
if cfg == "config2":
    sym = synth.text_bytes(100 << 20, synth.seed_for(2)); M = int(warps * sms * (waves or 3))
elif cfg == "config1":
    sym = synth.exp_bytes(1 << 20, 50, synth.seed_for(1, 50)); M = 16
else:
    sym = synth.exp_bytes(1 << 30, 50, synth.seed_for(3, 50)); M = int(warps * sms * (waves or 8))
f = R.recoil_build_model(synth.histogram(sym), 11)
c = R.recoil_encode(sym, f, 11, M) if kind == "recoil" else R.recoil_partitioned_encode(sym, f, 11, M)
dec = R.GpuDecoder(c, 0); dec.upload()
for _ in range(reps):
    dec.decode()
torch.cuda.synchronize()
assert dec.status()[0] == 0 and (dec.output().cpu().numpy() == sym).all()
print("ok", cfg, kind, M, len(c) / len(sym))
