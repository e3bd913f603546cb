cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python bench.py --no-cpu > gpurun_out/bench_c5_g22.json 2> gpurun_out/bench_c5_g22.err
timeout 900 python bench.py --config config2 --no-cpu --no-adaptive > gpurun_out/bench_c2_g22.json 2> gpurun_out/bench_c2_g22.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29519 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_mp2_g22.json 2> gpurun_out/bench_mp2_g22.err
python - <<'PY'
import json
for f in ["gpurun_out/bench_c5_g22.json", "gpurun_out/bench_c2_g22.json", "gpurun_out/bench_mp2_g22.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["bit_exact"], d.get("partitioned_baseline", {}).get("recoil_over_partitioned"),
              d.get("partitioned_same_encode"), d.get("config2_20k", {}).get("decoder_side_combine_to_half"))
    except Exception as e:
        print(f, "ERR", e)
PY
tail -3 gpurun_out/bench_mp2_g22.err
