cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for lib in nofixed fixed; do echo -n "$lib "; RECOIL_LIB=$PWD/build_var/v_$lib.so timeout 300 python tools/adaptive_timing.py; done; done > gpurun_out/ad_ab8.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_adaptive.py tests/test_gpu_decode.py -q -m gpu -k "adaptive or crafted or latent or random_models or coarse or for_device" > gpurun_out/pytest_ad8.log 2>&1
cat gpurun_out/ad_ab8.txt; tail -2 gpurun_out/pytest_ad8.log
