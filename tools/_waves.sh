cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for w in 1 1.25 1.5 1.75 2 3; do timeout 900 python bench.py --config config3 --waves $w --steps 20 --no-cpu --no-extra --no-adaptive 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config3 waves $w', d['config']['splits'], d['value'])"; done > gpurun_out/waves.txt 2>&1
timeout 900 python bench.py --config config4 --combine-to 2048 --steps 10 --no-cpu --no-adaptive > gpurun_out/cfg_c4_2048_extra.json 2>/dev/null
cat gpurun_out/waves.txt; python -c "import json; d=json.loads(open('gpurun_out/cfg_c4_2048_extra.json').read().strip().splitlines()[-1]); print('c4 2048', d['value'], d['partitioned_baseline'])"
