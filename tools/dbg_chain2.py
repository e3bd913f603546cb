import os, sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle
from paper_2306_12141_b200 import recoil as R
from test_gpu_adaptive import _random_models, _draw, gpu_decode_adaptive
N, n, K, M = 777777, 14, 40, 4096
rng = np.random.default_rng(N + n + K)
models = _random_models(rng, n, K)
sym, mid = _draw(rng, models, N, K)
c = R.recoil_encode_adaptive(sym, mid, models, n, M)
pts = oracle.container_points(c.tobytes())
ss = np.concatenate([[0], pts["sync_start"].astype(np.int64), [N]])
print("tasks", R.recoil_inspect(c)["n_splits"], "maxg", pts["maxg"][:5], "ss", ss[:6])
for rep in range(2):
    rc, bad, out, plan = gpu_decode_adaptive(c, mid)
    mism = np.nonzero(out != sym)[0]
    tasks = np.unique(np.searchsorted(ss, mism, side="right") - 1)
    print(os.environ.get("RECOIL_SCHED"), "rep", rep, "rc", rc, "mism", mism.size, "tasks", tasks[:12], len(tasks))
    for t in tasks[:3]:
        m = mism[(mism >= ss[t]) & (mism < ss[t + 1])]
        print("  task", t, "range", ss[t], ss[t + 1], "groups", ss[t] // 32, (ss[t + 1] - 1) // 32, "first", m[:8], "n", m.size,
              "start_group", pts["maxg"][t] if t < len(pts["maxg"]) else None)
