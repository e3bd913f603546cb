cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:recoil_decode_kernel -s 2 -c 1 -o gpurun_out/prof_adaptive_r2d python tools/profile_adaptive.py > /dev/null 2> gpurun_out/ncu_adaptive_r2d.err
ls -la gpurun_out/prof_adaptive_r2d.ncu-rep
