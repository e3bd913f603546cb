#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on small decodes
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cat > /tmp/san_case.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, synth, torch
from paper_2306_12141_b200 import recoil as R
ok = True
for kind, N, n, M, part in (("exp", 300000, 11, 64, False), ("text", 200000, 12, 100, True), ("image", 250000, 16, 20, False), ("exp", 1000, 11, 3, False)):
    sym = synth.workload(kind, N, seed=N, lam=40)
    f = R.recoil_build_model(synth.histogram(sym), n)
    c = R.recoil_partitioned_encode(sym, f, n, M) if part else R.recoil_encode(sym, f, n, M)
    for a, b in ((0, 1 << 64 - 1),) + ((tuple(R.recoil_shard_plan(c, 2)[:2]),) if not part else ()):
        dec = R.GpuDecoder(c, 0, a, b)
        dec.upload(); dec.decode(); rc, bad = dec.status()
        p = dec.plan
        out = dec.output().cpu().numpy()
        ok &= rc == 0 and bool((out == sym[p["out_lo"]:p["out_hi"]]).all())
        dec.close()
# adaptive codec (index-keyed models, 16-bit symbols)
lsym, mid, h = synth.latent_workload(150000, 4)
fm = np.concatenate([R.recoil_quantize(x, 16) for x in h["hist"]])
ca = R.recoil_encode_adaptive(lsym, mid, {"base": h["base"], "len": h["len"], "f": fm}, 16, 40)
for a, b in ((0, 1 << 64 - 1), tuple(R.recoil_shard_plan(ca, 2)[:2])):
    dec = R.GpuDecoder(ca, 0, a, b)
    dec.set_model_ids(mid)
    dec.upload(); dec.decode(); rc, bad = dec.status()
    p = dec.plan
    out = dec.output().cpu().numpy().view(np.uint16)
    ok &= rc == 0 and bool((out == lsym[p["out_lo"]:p["out_hi"]]).all())
    dec.close()
print("decodes ok" if ok else "DECODE MISMATCH")
PY
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_case.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "== $tool: $(tail -2 gpurun_out/sanitize_$tool.txt | tr '\n' ' ')"
done
