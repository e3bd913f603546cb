#!/bin/bash
# usage: tools/r2_bench.sh TAG -- new multi-device tests, default bench (config 5, 8 GiB), reference arm,
# config 3 with the size sweep, 2-rank strong-scaling run (both ranks on one GPU)
TAG=${1:-r2}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -m gpu > gpurun_out/pytest_multi_$TAG.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 1200 python bench.py --config config3 --size-sweep --no-adaptive > gpurun_out/bench_c3_$TAG.json 2> gpurun_out/bench_c3_$TAG.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_mp2_$TAG.json 2> gpurun_out/bench_mp2_$TAG.err
tail -n 3 gpurun_out/smoke_$TAG.log gpurun_out/pytest_multi_$TAG.log
for f in gpurun_out/bench_*_$TAG.json; do echo "== $f"; tail -c 1500 $f; echo; tail -3 ${f%.json}.err; done
