cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for lib in build_var/v_adold.so build_var/v_adnew.so; do RECOIL_LIB=$PWD/$lib timeout 300 python tools/adaptive_timing.py; done; done > gpurun_out/ad_ab.txt 2>&1
RECOIL_LIB=$PWD/build_var/v_adnew.so timeout 900 python -m pytest tests/test_gpu_adaptive.py -x -q -m gpu > gpurun_out/pytest_ad.log 2>&1
cat gpurun_out/ad_ab.txt; tail -3 gpurun_out/pytest_ad.log
