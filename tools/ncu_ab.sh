#!/bin/bash
# usage: tools/ncu_ab.sh TAG WAVES -- focused ncu metrics of the Recoil and partitioned decode at one
# split count (config 2 stream), for per-task overhead comparisons
TAG=${1:-ab}; WAVES=${2:-8}
cd "$(dirname "$0")/.." && mkdir -p gpurun_out
M="gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed_op_shfl.sum,smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_global_ld.sum,smsp__inst_executed_op_branch.sum"
for kind in recoil part; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:recoil_decode -s 1 -c 1 --csv python tools/profile_decode.py config2 $kind 2 $WAVES > gpurun_out/ncuab_${kind}_$TAG.csv 2> gpurun_out/ncuab_${kind}_$TAG.err
done
