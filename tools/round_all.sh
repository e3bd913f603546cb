#!/bin/bash
# usage: tools/round_all.sh TAG -- one GPU call for the round's evidence: smoke, full GPU tests, bench
# lines of every config (+ reference arm, 2-rank run), the ncu launch list of the default bench, one
# ncu --set full capture per config, compute-sanitizer
TAG=${1:-r}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 1500 python -m pytest tests/ -x -q -m gpu --durations=10 > gpurun_out/pytest_full_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu --no-adaptive > gpurun_out/bench_mp2_$TAG.json 2> gpurun_out/bench_mp2_$TAG.err
timeout 600 python bench.py --config config1 --steps 50 --no-extra > gpurun_out/bench_c1_$TAG.json 2> gpurun_out/bench_c1_$TAG.err
for lam in 10 50 200; do timeout 600 python bench.py --config config3 --lam $lam --steps 20 --no-extra --no-cpu > gpurun_out/bench_c3_l${lam}_$TAG.json 2> gpurun_out/bench_c3_l${lam}_$TAG.err; done
for tgt in 2048 256 16; do timeout 600 python bench.py --config config4 --combine-to $tgt --steps 10 --no-extra --no-cpu > gpurun_out/bench_c4_${tgt}_$TAG.json 2> gpurun_out/bench_c4_${tgt}_$TAG.err; done
timeout 900 python bench.py --config config5 --steps 10 --no-cpu > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-extra > /dev/null 2> gpurun_out/launches_$TAG.err
for cfg in config2 config1 config3 config5; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:recoil_decode -s 4 -c 1 -o gpurun_out/prof_${cfg}_$TAG python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu --no-extra > /dev/null 2> gpurun_out/ncu_${cfg}_$TAG.err
done
bash tools/sanitize.sh > gpurun_out/sanitize_summary_$TAG.txt 2>&1
tail -n 3 gpurun_out/smoke_$TAG.log gpurun_out/pytest_full_$TAG.log; cat gpurun_out/sanitize_summary_$TAG.txt
for f in gpurun_out/bench_*_$TAG.json; do echo "== $f"; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['unit'], d.get('bit_exact'), (d.get('roofline') or {}).get('frac'), d['config'].get('splits'), d.get('partitioned_baseline',{}).get('value'))" 2>&1 | tail -1; done
