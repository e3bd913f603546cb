#!/bin/bash
# usage: tools/r2_ranks.sh TAG -- the torchrun bench path with 4 and 8 ranks sharing one GPU (correctness
# of the strong-scaling setup: container hand-off, per-rank combine / shard / span regeneration / pinning)
TAG=${1:-r2r}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for n in 4 8; do
  timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench_mp${n}_$TAG.json 2> gpurun_out/bench_mp${n}_$TAG.err
  python -c "import json; d=json.loads(open('gpurun_out/bench_mp${n}_$TAG.json').read().strip().splitlines()[-1]); print($n, d['value'], d['bit_exact'], d['n_gpus'], d['scaling'], d['config']['splits'], d['e2e']['value'], d['setup_s'])" || tail -5 gpurun_out/bench_mp${n}_$TAG.err
done
