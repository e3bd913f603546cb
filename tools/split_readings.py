"""Compare the two readings of T in the split heuristic on the paper's
size-overhead setting (tab:overhead-n-11: 10 MB rand_lambda, 2176 splits, n = 11):
reading Z10' (T_m = ceil((N - prev - 1) / (M - m + 1)), the library's rule) vs
the printed T = ceil(N / M) fixed for every boundary.  Calls only oracle/.

usage: python tools/split_readings.py [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402

N, M, n = 10_000_000, 2176, 11
PAPER_KB = {10: 163.67, 50: 170.35, 100: 172.91, 200: 179.39, 500: 189.57}  # Recoil Large, n = 11


def main():
    out = {"N": N, "M_requested": M, "n": n, "rows": []}
    for lam in (10, 50, 200):
        sym = synth.exp_bytes(N, lam, synth.seed_for(3, lam))
        f = oracle.build_model(synth.histogram(sym), n)
        base = len(oracle.recoil_encode(sym, f, n, 1))
        row = {"dataset": f"rand_{lam}", "paper_recoil_large_kB": PAPER_KB[lam]}
        for name, pt in (("Z10_T_m", False), ("printed_T", True)):
            t0 = time.time()
            c = oracle.recoil_encode(sym, f, n, M, printed_T=pt)
            info = oracle.container_info(c)
            pts = oracle.container_points(c)
            bounds = np.concatenate([[0], pts["sync_start"].astype(np.int64), [N]])
            sizes = np.diff(bounds)
            row[name] = {"splits": info["M"], "overhead_kB": round((len(c) - base) / 1000, 2),
                         "task_symbols_max_over_mean": round(float(sizes.max() / sizes.mean()), 3),
                         "last_task_symbols": int(sizes[-1]), "seconds": round(time.time() - t0, 1)}
            print(lam, name, row[name], flush=True)
        out["rows"].append(row)
    path = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_split_readings.json"
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
