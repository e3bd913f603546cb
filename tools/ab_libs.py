"""Same-box A/B of kernel variants: python tools/ab_libs.py LIB1.so LIB2.so ...

Encodes each workload once (containers cached under /tmp), then times every library
in its own subprocess (RECOIL_LIB), alternating rounds, L2 flushed before every step,
CUDA events; prints the median decoded GB/s per (workload, lib) and checks bit-exactness.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WORKLOADS = [  # (name, kind, size, lam, splits)
    ("text100M_7104", "text", 100 << 20, 0, 7104),
    ("exp50_1G_10656", "exp", 1 << 30, 50, 10656),
    ("image_1G_10656", "image", 1 << 30, 0, 10656),
    ("text100M_21312", "text", 100 << 20, 0, 21312),
    ("text100M_10656", "text", 100 << 20, 0, 10656),
    ("text100M_14208", "text", 100 << 20, 0, 14208),
    ("exp50_1G_21312", "exp", 1 << 30, 50, 21312),
]
if os.environ.get("AB_WORKLOADS"):
    WORKLOADS = [w for w in WORKLOADS if w[0] in os.environ["AB_WORKLOADS"].split(",")]


def prepare():
    import numpy as np
    import synth
    from paper_2306_12141_b200 import recoil as R
    out = []
    for name, kind, n, lam, M in WORKLOADS:
        path = f"/tmp/ab_{name}.npy"
        part = f"/tmp/ab_{name}_part.npy"
        if not os.path.exists(path):
            sym = synth.workload(kind, n, seed=synth.seed_for(9, lam), lam=lam or 50)
            f = R.recoil_build_model(synth.histogram(sym), 11)
            np.save(path, R.recoil_encode(sym, f, 11, M))
            np.save(part, R.recoil_partitioned_encode(sym, f, 11, M))
            np.save(f"/tmp/ab_{name}_sym.npy", sym)
        out.append((name, path, part))
    return out


def time_one(container_path, sym_path, steps=20):
    import numpy as np
    import torch
    from paper_2306_12141_b200 import recoil as R
    c = np.load(container_path)
    sym = np.load(sym_path, mmap_mode="r")
    dec = R.GpuDecoder(c, 0)
    dec.upload()
    dec.decode()
    ok = dec.status()[0] == 0 and bool(torch.equal(dec.output(), torch.from_numpy(np.asarray(sym)).cuda()))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for _ in range(3):
        flush.fill_(1)
        dec.decode()
    for i in range(steps):
        flush.fill_(2)
        ev[i][0].record()
        dec.decode()
        ev[i][1].record()
    torch.cuda.synchronize()
    ms = float(np.median([a.elapsed_time(b) for a, b in ev]))
    n = len(sym)
    dec.close()
    return {"GBs": round(n / ms / 1e6, 1), "ms": round(ms, 4), "ok": ok}


def main():
    if sys.argv[1] == "--child":
        print(json.dumps(time_one(sys.argv[2], sys.argv[3])))
        return
    libs = sys.argv[1:]
    wl = prepare()
    rounds = int(os.environ.get("AB_ROUNDS", "3"))
    res = {}
    for r in range(rounds):
        for name, path, part in wl:
            for lib in libs + ["partitioned"]:
                env = dict(os.environ)
                if lib != "partitioned":
                    path_, *envs = lib.split(":")  # LIB.so[:VAR=VALUE...]
                    env["RECOIL_LIB"] = os.path.abspath(path_)
                    env.update(dict(e.split("=", 1) for e in envs))
                src = part if lib == "partitioned" else path
                p = subprocess.run([sys.executable, __file__, "--child", src, f"/tmp/ab_{name}_sym.npy"],
                                   env=env, capture_output=True, text=True)
                try:
                    d = json.loads(p.stdout.strip().splitlines()[-1])
                except Exception:
                    d = {"GBs": 0, "ok": False, "err": p.stderr[-400:]}
                res.setdefault((name, lib), []).append(d)
    for (name, lib), v in res.items():
        g = sorted(x["GBs"] for x in v)
        print(f"{name:18s} {os.path.basename(lib):40s} median {g[len(g) // 2]:8.1f} GB/s  all {g}  ok {all(x['ok'] for x in v)}",
              flush=True)


if __name__ == "__main__":
    main()
