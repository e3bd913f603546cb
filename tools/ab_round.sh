#!/bin/bash
# usage: tools/ab_round.sh TAG lib... -- A/B of library variants on the same box, alternating, 2 rounds
TAG=$1; shift
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for round in 1 2; do
for lib in default "$@"; do
  if [ "$lib" = default ]; then unset RECOIL_LIB; else export RECOIL_LIB=$PWD/$lib; fi
  for args in "--config config2 --waves 1" "--config config2 --waves 4" "--config config3 --waves 2" "--config config3 --waves 8"; do
    r=$(timeout 600 python bench.py $args --steps 20 --no-cpu --no-extra 2>/dev/null | tail -1)
    echo "$round $lib $args $(python -c "import json; d=json.loads('''$r'''); print(d['value'], d['bit_exact'], d['ms_per_step'], d['config']['splits'], d['clocks']['sm_mhz'])" 2>&1 | tail -1)"
  done
done
done | tee gpurun_out/ab_$TAG.txt
