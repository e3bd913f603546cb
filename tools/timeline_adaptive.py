"""Per-task timeline of one adaptive decode (variant build with -DRECOIL_TIMELINE via RECOIL_LIB).
usage: RECOIL_LIB=build_var/libtl.so AD_N=... python tools/timeline_adaptive.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2306_12141_b200 import recoil as R
N = int(os.environ.get("AD_N", 1 << 25))
sym, mid, h = synth.latent_workload(N, synth.seed_for(6))
f = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
K = len(h["len"])
warps, sms = R.recoil_decode_occupancy_adaptive(0, K, int(f.size))
c = R.recoil_encode_adaptive(sym, mid, {"base": h["base"], "len": h["len"], "f": f}, 16, warps * sms)
M = R.recoil_inspect(c)["n_splits"]
dec = R.GpuDecoder(c, 0)
dec.set_model_ids(mid)
dec.upload()
lib = R.load()
buf = np.zeros((M, 4), dtype=np.uint64)
scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(4):
    scratch.fill_(rep)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dec.decode(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
assert dec.status()[0] == 0
assert lib.recoil_timeline_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint32(M)) == 0
t0 = buf[:, 3].min()
ks, st, en = (buf[:, 3] - t0) / 1e3, (buf[:, 0] - t0) / 1e3, (buf[:, 1] - t0) / 1e3
dur = en - st
q = lambda a: " ".join(f"{np.percentile(a, p):8.2f}" for p in (0, 5, 25, 50, 75, 95, 100))
print(f"adaptive N={N} M={M} event ms={ms:.4f} span {en.max():.2f} us; percentiles 0/5/25/50/75/95/100")
print("warp kernel start  ", q(ks))
print("task start         ", q(st))
print("task duration      ", q(dur))
print("task end           ", q(en))
