cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do echo -n "nospan "; RECOIL_AD_NOSPAN=1 timeout 300 python tools/adaptive_timing.py; echo -n "span "; timeout 300 python tools/adaptive_timing.py; done > gpurun_out/ad_ab7.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_adaptive.py -q -m gpu > gpurun_out/pytest_ad7.log 2>&1
RECOIL_AD_NOSPAN=1 timeout 900 python -m pytest tests/test_gpu_adaptive.py -q -m gpu > gpurun_out/pytest_ad7n.log 2>&1
cat gpurun_out/ad_ab7.txt; tail -2 gpurun_out/pytest_ad7.log; tail -2 gpurun_out/pytest_ad7n.log
