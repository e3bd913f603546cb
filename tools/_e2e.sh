cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for ch in 8 16 32; do for st in 3 4; do timeout 900 python bench.py --config config3 --chunks $ch --streams $st --steps 10 --no-cpu --no-extra --no-adaptive 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks $ch streams $st', d['e2e']['value'], d['value'])"; done; done > gpurun_out/e2e_chunks.txt 2>&1
timeout 1200 python bench.py --chunks 16 --steps 10 --no-cpu --no-extra --no-adaptive 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('config5 chunks 16', d['e2e']['value'], d['value'], d.get('e2e_device_metadata',{}).get('value'))" >> gpurun_out/e2e_chunks.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_adaptive.py -q -m gpu > gpurun_out/pytest_ad_final.log 2>&1
cat gpurun_out/e2e_chunks.txt; tail -2 gpurun_out/pytest_ad_final.log
