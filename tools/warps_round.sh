#!/bin/bash
# usage: tools/warps_round.sh TAG -- warps-per-block variants: timing sweep + timelines (config 2 stream)
TAG=${1:-w}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
for v in default w16 w24 w32; do
  if [ "$v" = default ]; then unset RECOIL_LIB; TL=build_var/libtl.so; else export RECOIL_LIB=$PWD/build_var/lib$v.so; TL=build_var/libtl$v.so; fi
  echo "=== $v"; timeout 300 python tools/quick_timing.py 1,2,3 2>&1 | grep -v "^part"
  RECOIL_LIB=$PWD/$TL timeout 300 python tools/timeline.py text 100 1 2>&1 | grep "event\|task end\|occupancy\|block rank"
done
