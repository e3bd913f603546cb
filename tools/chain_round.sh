#!/bin/bash
# usage: tools/chain_round.sh TAG -- GPU tests (quick set) + waves sweep for config2/config3
TAG=${1:-r}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu -k "not 1GiB and not config3 and not config4" > gpurun_out/pytest_$TAG.log 2>&1
for args in "--config config2 --waves 1" "--config config2 --waves 2" "--config config2 --waves 4" "--config config2 --waves 8" "--config config3 --waves 2" "--config config3 --waves 8" "--config config3 --waves 32"; do
  r=$(timeout 600 python bench.py $args --steps 20 --no-cpu --no-extra 2>/dev/null | tail -1)
  echo "$args $(python -c "import json; d=json.loads('''$r'''); print(d['value'], d['bit_exact'], d['ms_per_step'], d['config']['splits'])" 2>&1 | tail -1)"
done | tee gpurun_out/chain_$TAG.txt
tail -n 3 gpurun_out/smoke_$TAG.log gpurun_out/pytest_$TAG.log
