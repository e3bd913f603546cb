cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for lib in v_adu16 v_adu4 v_adl2 v_adl4 v_adl16; do echo -n "$lib "; RECOIL_LIB=$PWD/build_var/$lib.so timeout 300 python tools/adaptive_timing.py; done; done > gpurun_out/ad_ab2.txt 2>&1
cat gpurun_out/ad_ab2.txt
