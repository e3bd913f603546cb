#!/bin/bash
# usage: tools/e2e_sweep.sh TAG -- e2e pipeline chunk / stream sweep (config 2)
TAG=${1:-r}; export TAG
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cs in ${E2E_SWEEP:-"4 2" "8 2" "8 3" "16 3" "16 4" "32 4"}; do
  set -- $cs
  timeout 300 python bench.py --steps 10 --no-cpu --no-extra --chunks $1 --streams $2 2>/dev/null | tail -1 > gpurun_out/e2e_$TAG.json
  python - "$1" "$2" <<'PY'
import json, sys
d = json.loads(open(sys.argv[0] if False else "gpurun_out/e2e_" + __import__("os").environ.get("TAG", "r") + ".json").read())
print("chunks", sys.argv[1], "streams", sys.argv[2], d["value"], d["e2e"]["value"])
PY
done | tee gpurun_out/e2e_sweep_$TAG.txt
