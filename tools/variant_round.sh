#!/bin/bash
# usage: tools/variant_round.sh TAG lib1.so lib2.so ... -- bench config2 + config3 per library variant
TAG=$1; shift
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for lib in default "$@"; do
  if [ "$lib" = default ]; then unset RECOIL_LIB; else export RECOIL_LIB=$PWD/$lib; fi
  for cfg in config2 config3; do
    r=$(timeout 600 python bench.py --config $cfg --steps 20 --no-cpu --no-extra 2>/dev/null | tail -1)
    echo "$lib $cfg $(python -c "import json; d=json.loads('''$r'''); print(d['value'], d['bit_exact'], d['ms_per_step'], d['config']['splits'])" 2>&1 | tail -1)"
  done
done | tee gpurun_out/variants_$TAG.txt
