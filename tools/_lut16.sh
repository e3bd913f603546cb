cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
RECOIL_LIB=$PWD/build_var/v_lut16.so timeout 900 python -m pytest tests/test_gpu_decode.py -x -q -m gpu -k "not 8GiB and not 2pow31 and not config3 and not config4" > gpurun_out/pytest_lut16.log 2>&1
tail -2 gpurun_out/pytest_lut16.log
AB_ROUNDS=3 timeout 1500 python tools/ab_libs.py build_var/v_base.so build_var/v_lut16.so > gpurun_out/ab_lut16.txt 2>&1
cat gpurun_out/ab_lut16.txt
