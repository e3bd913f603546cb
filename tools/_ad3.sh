cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do echo -n "v1 "; RECOIL_AD_V1=1 timeout 300 python tools/adaptive_timing.py; echo -n "v2 "; timeout 300 python tools/adaptive_timing.py; done > gpurun_out/ad_ab3.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_adaptive.py -q -m gpu > gpurun_out/pytest_ad3.log 2>&1
RECOIL_AD_V1=1 timeout 900 python -m pytest tests/test_gpu_adaptive.py -q -m gpu > gpurun_out/pytest_ad3v1.log 2>&1
cat gpurun_out/ad_ab3.txt; tail -3 gpurun_out/pytest_ad3.log; tail -3 gpurun_out/pytest_ad3v1.log
