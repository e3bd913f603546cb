#!/bin/bash
# usage: tools/r2_evidence.sh TAG -- round-2 evidence in one GPU call: device-meta tests, the default bench
# (config 5, 8 GiB), the reference arm, a 2-rank strong-scaling run (both ranks on one GPU), the ncu launch
# list of the default bench, ncu --set full of one decode launch for config 5 and config 3
TAG=${1:-r2}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_device_meta.py tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_dm_$TAG.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_mp2_$TAG.json 2> gpurun_out/bench_mp2_$TAG.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2> gpurun_out/launches_$TAG.err
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:recoil_decode_kernel -s 4 -c 1 -o gpurun_out/prof_config5_$TAG python bench.py --steps 3 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2> gpurun_out/ncu_config5_$TAG.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recoil_decode_kernel -s 4 -c 1 -o gpurun_out/prof_config3_$TAG python bench.py --config config3 --steps 3 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2> gpurun_out/ncu_config3_$TAG.err
tail -n 3 gpurun_out/smoke_$TAG.log gpurun_out/pytest_dm_$TAG.log
for f in gpurun_out/bench_*_$TAG.json; do echo "== $f"; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['unit'], d.get('bit_exact'), (d.get('roofline') or {}).get('frac'), d['config'].get('splits'), d.get('partitioned_baseline',{}).get('recoil_over_partitioned'), d.get('e2e'))" 2>&1 | tail -1; tail -2 ${f%.json}.err; done
ls -la gpurun_out/*$TAG*
