cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:recoil_decode_kernel -s 4 -c 1 -o gpurun_out/prof_config1_r2e python bench.py --config config1 --steps 3 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:recoil_decode_kernel -s 4 -c 1 -o gpurun_out/prof_config2_r2e python bench.py --config config2 --steps 3 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2>&1
for t in 2048 256 16; do timeout 900 ncu --set full --clock-control none -k regex:recoil_decode_kernel -s 4 -c 1 -o gpurun_out/prof_config4_${t}_r2e python bench.py --config config4 --combine-to $t --steps 3 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2>&1; done
ls gpurun_out/*r2e*
