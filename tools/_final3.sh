cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_f3.log 2>&1
timeout 2400 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_all_f3.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench_c5_f3.json 2> gpurun_out/bench_c5_f3.err
tail -3 gpurun_out/smoke_f3.log; tail -4 gpurun_out/pytest_all_f3.log
python -c "import json; d=json.loads(open('gpurun_out/bench_c5_f3.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['partitioned_baseline']['recoil_over_partitioned'], d.get('partitioned_same_encode',{}).get('recoil_over_partitioned'), d['adaptive_latent']['symbols_per_s']/1e9, d.get('e2e_device_metadata',{}).get('value'), d.get('device_combine'), d['roofline']['frac'], d['clocks'])"
