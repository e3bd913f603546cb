"""Library vs oracle on the full-size configs ("the large configs compare SHA-256 of
the containers"): the same synthetic stream encoded by recoil_encode (librecoil) and by the oracle
(or_recoil_encode, plain C), byte-identical containers.  CPU only; minutes per GiB.
usage: python tools/host_parity_large.py > profiles/r02_host_parity_large.txt"""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2306_12141_b200 import recoil as R  # noqa: E402

CASES = [("config2 100 MiB text, 10656 splits", "text", 100 << 20, 0, 2, 10656),
         ("config3 1 GiB exp lambda=50, 10656 splits", "exp", 1 << 30, 50, 3, 10656),
         ("config1 1 MiB exp lambda=50, 16 splits", "exp", 1 << 20, 50, 1, 16)]
for name, kind, n, lam, cfg, M in CASES:
    sym = synth.workload(kind, n, seed=synth.seed_for(cfg, lam), lam=lam or 50)
    f = R.recoil_build_model(synth.histogram(sym), 11)
    fo = oracle.build_model(synth.histogram(sym), 11)
    assert (f == fo).all(), name
    t0 = time.time()
    c = R.recoil_encode(sym, f, 11, M)
    t1 = time.time()
    co = oracle.recoil_encode(sym, fo, 11, M)
    t2 = time.time()
    h1, h2 = hashlib.sha256(c.tobytes()).hexdigest(), hashlib.sha256(co).hexdigest()
    print(f"{name}: library {len(c)} B sha256 {h1[:16]} ({t1 - t0:.1f} s), oracle {len(co)} B sha256 {h2[:16]} "
          f"({t2 - t1:.1f} s): {'IDENTICAL' if h1 == h2 else 'DIFFERENT'}", flush=True)
    assert h1 == h2
