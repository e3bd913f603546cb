cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in 1 2; do for lib in v_adw32 v_adw24 v_adw16; do echo -n "$lib "; RECOIL_LIB=$PWD/build_var/$lib.so timeout 300 python tools/adaptive_timing.py; done; done > gpurun_out/ad_w.txt 2>&1
cat gpurun_out/ad_w.txt
