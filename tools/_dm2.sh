cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_device_meta.py -q -m gpu > gpurun_out/pytest_dm2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/dm2_launches.csv python bench.py --config config3 --steps 3 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2>&1
tail -3 gpurun_out/pytest_dm2.log; grep -E "k_spec|k_write|k_resolve|k_global|k_lut|k_taskrecs" gpurun_out/dm2_launches.csv | awk -F'","' '{print $5, $(NF)}' | sort | uniq -c | head -20
