"""Per-task timeline of one decode (variant build with -DRECOIL_TIMELINE, loaded via RECOIL_LIB).
usage: RECOIL_LIB=build_var/libtl.so python tools/timeline.py [text|exp] [MiB] [waves]"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2306_12141_b200 import recoil as R
kind = sys.argv[1] if len(sys.argv) > 1 else "text"
mib = int(sys.argv[2]) if len(sys.argv) > 2 else 100
waves = float(sys.argv[3]) if len(sys.argv) > 3 else 1
warps, sms = R.recoil_decode_occupancy(0, 11)
sym = synth.text_bytes(mib << 20, synth.seed_for(2)) if kind == "text" else synth.exp_bytes(mib << 20, 50, synth.seed_for(3, 50))
f = R.recoil_build_model(synth.histogram(sym), 11)
c = R.recoil_encode(sym, f, 11, int(warps * sms * waves))
M = R.recoil_inspect(c)["n_splits"]
dec = R.GpuDecoder(c, 0); dec.upload()
lib = R.load()
buf = np.zeros((M, 4), dtype=np.uint64)
scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for rep in range(4):
    scratch.fill_(rep)  # L2 flush as in bench.py
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dec.decode(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
assert dec.status()[0] == 0 and (dec.output().cpu().numpy() == sym).all()
assert lib.recoil_timeline_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint32(M)) == 0
t0 = buf[:, 3].min()
ks, st, en = (buf[:, 3] - t0) / 1e3, (buf[:, 0] - t0) / 1e3, (buf[:, 1] - t0) / 1e3
sm = (buf[:, 2] & 0xFFFF).astype(int)
dur = en - st
print(f"{kind} {mib} MiB waves={waves} M={M} event ms={ms:.4f}  span(first warp start -> last task end) {en.max():.2f} us")
q = lambda a: " ".join(f"{np.percentile(a, p):7.2f}" for p in (0, 5, 25, 50, 75, 95, 100))
print("percentiles 0/5/25/50/75/95/100")
print("warp kernel start  ", q(ks))
print("first-task start   ", q(st[st <= np.sort(st)[min(len(st)-1, warps*sms-1)]]))
print("task duration      ", q(dur))
print("task end           ", q(en))
sm_end = np.array([en[sm == s].max() for s in np.unique(sm)])
sm_mean_end = np.array([en[sm == s].mean() for s in np.unique(sm)])
print("per-SM last end    ", q(sm_end))
print("per-SM mean end    ", q(sm_mean_end))
busy = dur.sum() / (len(np.unique(sm)) * warps * en.max())
print(f"warp-slot occupancy over the span: {busy:.3f}")
# unfairness structure (first-wave tasks: one per warp slot)
gw = (buf[:, 2] >> 16).astype(np.int64)
first = np.zeros(len(gw), bool)
seen = set()
for i in np.argsort(st):
    if gw[i] not in seen:
        seen.add(gw[i]); first[i] = True
wpb = int(os.environ.get("WPB", "24"))  # warps per block of the build
blk, wib = gw // wpb, gw % wpb
print("mean first-task duration by warp-in-block:", " ".join(f"{dur[first & (wib == k)].mean():6.1f}" for k in range(wpb)))
rank = np.zeros(len(gw), int)
for s in np.unique(sm):
    bl = np.unique(blk[sm == s])
    for r, b in enumerate(bl):
        rank[(sm == s) & (blk == b)] = r
print("mean first-task duration by block rank on its SM:", " ".join(f"{dur[first & (rank == k)].mean():6.1f}" for k in range(rank.max() + 1)))
print("mean first-task duration by SMSP (warp-in-block % 4):", " ".join(f"{dur[first & (wib % 4 == k)].mean():6.1f}" for k in range(4)))
b2 = blk
rows = {}
for i in range(len(gw)):
    rows.setdefault(int(b2[i]), int(sm[i]))
bl = sorted(rows)
print("block -> SM (first 12):", [(b, rows[b]) for b in bl[:12]])
print("block -> SM (148..159):", [(b, rows[b]) for b in bl[148:160]])
persm = {}
for b in bl:
    persm.setdefault(rows[b], []).append(b)
print("SM -> blocks (first 6 SMs):", [(s, persm[s]) for s in sorted(persm)[:6]])
