cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
RECOIL_LIB=$PWD/build_var/v_regstage.so timeout 900 python -m pytest tests/test_gpu_decode.py -x -q -m gpu -k "not 8GiB and not 2pow31" > gpurun_out/pytest_regstage.log 2>&1
tail -3 gpurun_out/pytest_regstage.log
timeout 1500 python tools/ab_libs.py build_var/v_base.so build_var/v_base.so:RECOIL_PLAN_PREBUILT=1 build_var/v_regstage.so build_var/v_regstage.so:RECOIL_PLAN_PREBUILT=1 > gpurun_out/ab_regstage.txt 2>&1
cat gpurun_out/ab_regstage.txt | tail -20
