"""e2e pipeline probe: host enqueue time vs total, and raw PCIe copy rates on this box."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2306_12141_b200 import recoil as R
sym = synth.text_bytes(100 << 20, synth.seed_for(2))
f = R.recoil_build_model(synth.histogram(sym), 11)
w, s = R.recoil_decode_occupancy(0, 11)
c = R.recoil_encode(sym, f, 11, w * s)
pinned = torch.empty(len(c), dtype=torch.uint8, pin_memory=True); pinned.numpy()[:] = c
out = torch.empty(len(sym), dtype=torch.uint8, pin_memory=True)
for chunks, streams in ((8, 3), (4, 2), (2, 2), (1, 1)):
    pipe = R.HostPipeline(pinned.numpy(), 0, n_chunks=chunks, n_streams=streams)
    enq, tot = [], []
    for i in range(8):
        torch.cuda.synchronize()
        t0 = time.perf_counter(); pipe.run(out); t1 = time.perf_counter(); rc, _ = pipe.status(); t2 = time.perf_counter()
        enq.append(t1 - t0); tot.append(t2 - t0)
    print(f"chunks {chunks} streams {streams}: enqueue {1e3*np.median(enq):.3f} ms total {1e3*np.median(tot):.3f} ms e2e {len(sym)/np.median(tot)/1e9:.1f} GB/s ok={rc==0 and (out.numpy()==sym).all()}")
    pipe.close()
# raw copy rates
d = torch.empty(len(sym), dtype=torch.uint8, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(out, non_blocking=True)), ("D2H", lambda: out.copy_(d, non_blocking=True))):
    ts = []
    for i in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(name, f"{len(sym)/np.median(ts)/1e9:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
h2 = torch.empty(len(sym), dtype=torch.uint8, pin_memory=True); d2 = torch.empty_like(d)
ts = []
for i in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(out, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("H2D||D2H", f"{2*len(sym)/np.median(ts)/1e9:.1f} GB/s total")
