cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_g5.log 2>&1
timeout 600 python -m pytest tests/test_gpu_device_meta.py -x -q -m gpu > gpurun_out/pytest_dm_g5.log 2>&1
timeout 1800 python -m pytest tests/ -x -q -m gpu --durations=8 > gpurun_out/pytest_all_g5.log 2>&1
timeout 900 python bench.py --config config3 --no-adaptive > gpurun_out/bench_c3_g5.json 2> gpurun_out/bench_c3_g5.err
tail -3 gpurun_out/smoke_g5.log; tail -15 gpurun_out/pytest_dm_g5.log; tail -12 gpurun_out/pytest_all_g5.log; tail -c 2500 gpurun_out/bench_c3_g5.json; tail -3 gpurun_out/bench_c3_g5.err
