#!/bin/bash
TAG=$1
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for args in "--config config3 --waves 2" "--config config3 --waves 4" "--config config3 --waves 8" "--config config3 --waves 16" "--config config2 --waves 4" "--config config2 --waves 8"; do
  r=$(timeout 600 python bench.py $args --steps 10 --no-cpu --no-extra 2>/dev/null | tail -1)
  echo "$args $(python -c "import json; d=json.loads('''$r'''); print(d['value'], d['bit_exact'], d['ms_per_step'], d['config']['splits'])" 2>&1 | tail -1)"
done | tee gpurun_out/waves_$TAG.txt
