#!/bin/bash
# usage: tools/gpu_round.sh TAG [pytest-k-expr] [ncu]
TAG=${1:-run}; KEXPR=${2:-"not 1GiB and not config3 and not config4"}; NCU=${3:-}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python tools/quick_timing.py > gpurun_out/quick_$TAG.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_decode.py -x -q -m gpu -k "$KEXPR" > gpurun_out/pytest_$TAG.log 2>&1
if [ -n "$NCU" ]; then
  ncu --set full --clock-control none --import-source on -k regex:recoil_decode -s 1 -c 1 -o gpurun_out/prof_$TAG python tools/profile_decode.py config2 recoil 2 > gpurun_out/ncu_$TAG.log 2>&1
fi
tail -2 gpurun_out/smoke_$TAG.log; cat gpurun_out/quick_$TAG.log; tail -3 gpurun_out/pytest_$TAG.log
