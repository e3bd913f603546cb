cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_device_meta.py tests/test_gpu_multi.py -q -m gpu > gpurun_out/pytest_dm_g6.log 2>&1
timeout 1800 python -m pytest tests/ -q -m gpu --durations=5 --deselect tests/test_gpu_decode.py::test_config5_8GiB_full_size_sharded > gpurun_out/pytest_all_g6.log 2>&1
tail -25 gpurun_out/pytest_dm_g6.log; tail -12 gpurun_out/pytest_all_g6.log
