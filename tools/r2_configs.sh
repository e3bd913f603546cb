#!/bin/bash
# usage: tools/r2_configs.sh TAG -- bench lines of every BASELINE config on the current build, compute-sanitizer
# on the round-2 GPU code (device metadata path, multi-device decode), ncu source-level capture of the adaptive kernel
TAG=${1:-r2c}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --config config1 --steps 50 --no-extra > gpurun_out/cfg_c1_$TAG.json 2> gpurun_out/cfg_c1_$TAG.err
timeout 900 python bench.py --config config2 --no-adaptive > gpurun_out/cfg_c2_$TAG.json 2> gpurun_out/cfg_c2_$TAG.err
for lam in 10 100 200; do timeout 600 python bench.py --config config3 --lam $lam --steps 20 --no-cpu --no-adaptive > gpurun_out/cfg_c3_l${lam}_$TAG.json 2> gpurun_out/cfg_c3_l${lam}_$TAG.err; done
for tgt in 2048 256 16; do timeout 600 python bench.py --config config4 --combine-to $tgt --steps 10 --no-cpu --no-extra > gpurun_out/cfg_c4_${tgt}_$TAG.json 2> gpurun_out/cfg_c4_${tgt}_$TAG.err; done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_device_meta.py tests/test_gpu_multi.py -q -m gpu -k "not 65536 and not config4" > gpurun_out/san_memcheck_$TAG.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san_memcheck_$TAG.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_device_meta.py -q -m gpu -k "bit_exact or combine_equals" > gpurun_out/san_racecheck_$TAG.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san_racecheck_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recoil_decode_kernel -s 2 -c 1 -o gpurun_out/prof_adaptive_$TAG python tools/profile_adaptive.py > /dev/null 2> gpurun_out/ncu_adaptive_$TAG.err
for f in gpurun_out/cfg_*_$TAG.json; do echo "== $f"; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['unit'], d.get('bit_exact'), (d.get('roofline') or {}).get('frac'), d['config'].get('splits'), (d.get('partitioned_baseline') or {}).get('recoil_over_partitioned'), (d.get('config2_20k') or {}).get('recoil_over_partitioned'))" 2>&1 | tail -1; done
tail -3 gpurun_out/san_memcheck_$TAG.log gpurun_out/san_racecheck_$TAG.log
