"""Compressed-size overhead vs split count (BASELINE metric, second half; paper
tab:overhead-n-11 / tab:overhead-n-16), on the synthetic stand-ins of
the paper's datasets, through the library (host only).

Variants: (a) one codec (M = 1), (b) Conventional Large = 2176
partitions, (c) Recoil Large = 2176 splits, (d) Conventional Small = 16
partitions (re-encoded), (e) Recoil Small = (c) combined to 16 splits.
Overheads are bytes over (a); 1 KB = 1000 B as in the paper.

usage: python tools/size_overhead.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_2306_12141_b200 import recoil as R  # noqa: E402

PAPER = {  # (b), (c), (d), (e) in KB, n = 11 / n = 16
    11: {"rand_10": (211.44, 163.67, 1.47, 1.12), "rand_50": (211.37, 170.35, 1.45, 1.16),
         "rand_100": (211.25, 172.91, 1.45, 1.18), "rand_200": (211.32, 179.39, 1.27, 1.09),
         "rand_500": (203.31, 189.57, 1.27, 1.14), "enwik8": (212.70, 165.56, 1.45, 1.12)},
    16: {"rand_10": (211.19, 163.94, 1.47, 1.12), "rand_50": (210.56, 171.53, 1.47, 1.15),
         "rand_100": (211.03, 172.10, 1.46, 1.17), "rand_200": (208.95, 180.90, 1.30, 1.09),
         "rand_500": (208.53, 190.75, 1.27, 1.14), "enwik8": (212.35, 165.28, 1.47, 1.12),
         "div2k801": (215.75, 173.41, 1.46, 1.18)},
}
N = 10_000_000  # the rand_* datasets are 10 MB


def static_row(sym, n):
    f = R.recoil_build_model(synth.histogram(sym), n)
    a = len(R.recoil_encode(sym, f, n, 1))
    b = len(R.recoil_partitioned_encode(sym, f, n, 2176)) - len(R.recoil_partitioned_encode(sym, f, n, 1))
    big = R.recoil_encode(sym, f, n, 2176)
    c = len(big) - a
    d = len(R.recoil_partitioned_encode(sym, f, n, 16)) - len(R.recoil_partitioned_encode(sym, f, n, 1))
    e = len(R.recoil_combine_splits(big, 16)) - a
    return {"baseline_bytes": a, "splits_large": R.recoil_inspect(big)["n_splits"],
            "conv_large": b, "recoil_large": c, "conv_small": d, "recoil_small": e}


def main():
    rows = {}
    for n in (11, 16):
        for lam in (10, 50, 100, 200, 500):
            rows[f"n{n}/rand_{lam}"] = static_row(synth.exp_bytes(N, lam, synth.seed_for(3, lam)), n)
        rows[f"n{n}/enwik8-like"] = static_row(synth.text_bytes(N, synth.seed_for(2)), n)
        rows[f"n{n}/image-residual"] = static_row(synth.image_bytes(N, synth.seed_for(5)), n)
    # div2k stand-in: 16-bit latent symbols with index-keyed Gaussian models (adaptive), n = 16
    sym, mid, h = synth.latent_workload(3_600_000, synth.seed_for(6))  # div2k801: 7,209 KB of 16-bit symbols
    f = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
    models = {"base": h["base"], "len": h["len"], "f": f}
    a = len(R.recoil_encode_adaptive(sym, mid, models, 16, 1))
    big = R.recoil_encode_adaptive(sym, mid, models, 16, 2176)
    rows["n16/latent (div2k-like, adaptive)"] = {
        "baseline_bytes": a, "splits_large": R.recoil_inspect(big)["n_splits"], "conv_large": None,
        "recoil_large": len(big) - a, "conv_small": None, "recoil_small": len(R.recoil_combine_splits(big, 16)) - a}
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                              "r01_size_overhead.json")
    json.dump({"note": __doc__.strip().splitlines()[0], "paper_KB": PAPER, "rows": rows}, open(out, "w"), indent=1)
    print(f"| dataset | splits | (b) conv large KB | (c) recoil large KB | (d) conv small KB | (e) recoil small KB | paper (b)/(c)/(d)/(e) |")
    print("|---|---|---|---|---|---|---|")
    for k, r in rows.items():
        n = int(k[1:3])
        name = k.split("/")[1].split(" ")[0].replace("-like", "")
        pname = {"enwik8": "enwik8", "latent": "div2k801"}.get(name, name)
        p = PAPER.get(n, {}).get(pname)
        kb = lambda v: "N/A" if v is None else f"{v / 1000:.2f}"
        print(f"| {k} | {r['splits_large']} | {kb(r['conv_large'])} | {kb(r['recoil_large'])} | {kb(r['conv_small'])} | "
              f"{kb(r['recoil_small'])} | {'/'.join(str(x) for x in p) if p else '-'} |")


if __name__ == "__main__":
    main()
