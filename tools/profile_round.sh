#!/bin/bash
# usage: tools/profile_round.sh TAG -- bench lines (default + reference arm), ncu launch list of the
# default bench command, one ncu --set full capture of the decode kernel per config
TAG=${1:-r}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-extra > /dev/null 2> gpurun_out/launches_$TAG.err
for cfg in config2 config1 config3 config5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:recoil_decode -s 4 -c 1 -o gpurun_out/prof_${cfg}_$TAG python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-extra > /dev/null 2> gpurun_out/ncu_${cfg}_$TAG.err
done
cat gpurun_out/bench_$TAG.json gpurun_out/bench_ref_$TAG.json; tail -3 gpurun_out/bench_$TAG.err
