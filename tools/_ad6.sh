cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for lib in base first clamp both; do echo -n "$lib "; RECOIL_LIB=$PWD/build_var/v_ad_$lib.so timeout 300 python tools/adaptive_timing.py; done; done > gpurun_out/ad_ab6.txt 2>&1
RECOIL_LIB=$PWD/build_var/v_ad_both.so timeout 900 python -m pytest tests/test_gpu_adaptive.py -q -m gpu > gpurun_out/pytest_ad6.log 2>&1
cat gpurun_out/ad_ab6.txt; tail -2 gpurun_out/pytest_ad6.log
