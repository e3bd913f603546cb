cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for lib in v_adu16 v_adu4 v_adl4 v_adl16; do echo "== $lib"; RECOIL_LIB=$PWD/build_var/$lib.so timeout 300 python -m pytest tests/test_gpu_adaptive.py -q -m gpu -x -k "random_models" 2>&1 | tail -2; done > gpurun_out/ad_iso.txt 2>&1
echo "== tree"; timeout 300 python -m pytest tests/test_gpu_adaptive.py -q -m gpu -x -k "random_models" 2>&1 | tail -2 >> gpurun_out/ad_iso.txt
cat gpurun_out/ad_iso.txt
