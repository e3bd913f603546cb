import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle, synth
from paper_2306_12141_b200 import recoil as R
from test_gpu_adaptive import _random_models, _draw, gpu_decode_adaptive
N, n, K, M = 1 << 20, 16, 200, 2176
rng = np.random.default_rng(N + n + K)
models = _random_models(rng, n, K)
sym, mid = _draw(rng, models, N, K)
c = R.recoil_encode_adaptive(sym, mid, models, n, M)
pts = oracle.container_points(c.tobytes())
ss = np.concatenate([[0], pts["sync_start"].astype(np.int64), [N]])
for rep in range(3):
    rc, bad, out, plan = gpu_decode_adaptive(c, mid)
    mism = np.nonzero(out != sym)[0]
    tasks = np.unique(np.searchsorted(ss, mism, side="right") - 1)
    print("adaptive rep", rep, "rc", rc, "mism", mism.size, "tasks", tasks[:20], len(tasks))
# static with the same geometry
sym8 = synth.exp_bytes(N, 50, 5)
f = R.recoil_build_model(synth.histogram(sym8), 11)
for Ms in (2176, 7104 * 4, 100000):
    c8 = R.recoil_encode(sym8, f, 11, Ms)
    pts8 = oracle.container_points(c8.tobytes())
    ss8 = np.concatenate([[0], pts8["sync_start"].astype(np.int64), [N]])
    dec = R.GpuDecoder(c8, 0); dec.upload()
    for rep in range(3):
        dec.decode(); rc, bad = dec.status(); out = dec.output().cpu().numpy()
        mism = np.nonzero(out != sym8)[0]
        tasks = np.unique(np.searchsorted(ss8, mism, side="right") - 1)
        print("static M", Ms, "rep", rep, "rc", rc, "mism", mism.size, "tasks", tasks[:10], len(tasks))
    dec.close()
