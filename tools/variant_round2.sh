#!/bin/bash
TAG=$1; shift
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for lib in "$@"; do
  export RECOIL_LIB=$PWD/$lib
  for args in "--config config2 --waves 1" "--config config2 --waves 2" "--config config2 --waves 3" "--config config3" "--config config5"; do
    r=$(timeout 600 python bench.py $args --steps 20 --no-cpu --no-extra 2>/dev/null | tail -1)
    echo "$lib $args $(python -c "import json; d=json.loads('''$r'''); print(d['value'], d['bit_exact'], d['ms_per_step'], d['config']['splits'])" 2>&1 | tail -1)"
  done
done | tee gpurun_out/variants_$TAG.txt
