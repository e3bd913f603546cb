cd $GRAFT_REPO_ROOT && mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:recoil_decode_kernel -s 4 -c 1 -o /tmp/prof_config1_r2e python bench.py --config config1 --steps 3 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:recoil_decode_kernel -s 4 -c 1 -o /tmp/prof_config2_r2e python bench.py --config config2 --steps 3 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2>&1
for t in 2048 256 16; do timeout 900 ncu --set full --clock-control none -k regex:recoil_decode_kernel -s 4 -c 1 -o /tmp/prof_config4_${t}_r2e python bench.py --config config4 --combine-to $t --steps 3 --warmup 3 --no-cpu --no-extra --no-adaptive > /dev/null 2>&1; done
python - <<'PY'
import json, sys, os
sys.path.insert(0, "tools")
import refresh_profiles as rp
for name in ["config1", "config2", "config4_2048", "config4_256", "config4_16"]:
    rep = f"/tmp/prof_{name}_r2e.ncu-rep"
    if os.path.exists(rep):
        json.dump(rp.summary(rep), open(f"gpurun_out/sum_{name}_r2e.json", "w"), indent=1)
        print(name, "ok")
PY
ls -la gpurun_out/
