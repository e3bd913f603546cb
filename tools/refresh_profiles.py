"""Turn ncu --set full captures (gpurun_out/prof_<config>_<tag>.ncu-rep) into the
committed summaries under profiles/ and the per-launch numbers bench.py reads
(profiles/ncu_traffic.json): DRAM bytes and shared-memory wavefronts per launch.

usage: python tools/refresh_profiles.py [--round=r02] TAG config5:10656 config3:10656 ...
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__maximum_warps_per_active_cycle_pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__cycles_active.avg", "sm__cycles_elapsed.avg.per_second", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed.sum", "launch__shared_mem_per_block_static",
        "smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
        "smsp__average_warp_latency_issue_stalled_wait.ratio",
        "smsp__average_warp_latency_issue_stalled_not_selected.ratio",
        "smsp__average_warp_latency_issue_stalled_mio_throttle.ratio",
        "smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio",
        "smsp__average_warp_latency_issue_stalled_lg_throttle.ratio",
        "smsp__average_warp_latency_issue_stalled_selected.ratio",
        "smsp__average_warp_latency_issue_stalled_barrier.ratio",
        "smsp__average_warp_latency_issue_stalled_membar.ratio",
        "smsp__average_warp_latency_issue_stalled_branch_resolving.ratio",
        "smsp__average_warp_latency_issue_stalled_dispatch_stall.ratio",
        "smsp__average_warp_latency_issue_stalled_no_instruction.ratio",
        "smsp__average_warp_latency_issue_stalled_drain.ratio",
        "smsp__average_warp_latency_issue_stalled_sleeping.ratio",
        "smsp__warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__warps_issue_stalled_selected_per_issue_active.ratio",
        "smsp__inst_executed_op_shared_ld.sum", "smsp__inst_executed_op_shared_st.sum",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__mio_inst_issued.avg.pct_of_peak_sustained_active", "sm__mio_pq_read_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__mio2rf_writeback_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_issued.avg.per_cycle_active", "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_cbu.avg.pct_of_peak_sustained_active"]


def summary(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else None}
    for w in WANT:
        if w in hdr:
            i = hdr.index(w)
            v = vals[i].replace(",", "")
            try:
                v = float(v)
            except ValueError:
                pass
            out[w] = {"value": v, "unit": units[i]}
    return out


def main():
    rnd = "r02"
    if sys.argv[1].startswith("--round="):
        rnd = sys.argv.pop(1).split("=", 1)[1]
    tag = sys.argv[1]
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(tf)) if os.path.exists(tf) else {}
    for spec in sys.argv[2:]:
        # "config3:14208", or "config4@2048:2048" for a capture named prof_config4_2048_<tag>
        cfgv, M = spec.split(":")
        cfg, _, var = cfgv.partition("@")
        name = f"{cfg}_{var}" if var else cfg
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{name}_{tag}.ncu-rep")
        s = summary(rep)
        s["source"] = f"ncu --set full --clock-control none, 1 decode launch of bench.py --config {cfg} ({M} splits)"
        dst = os.path.join(ROOT, "profiles", f"{rnd}_decode_{name}_ncu_full.json")
        json.dump(s, open(dst, "w"), indent=1)
        rd = s["dram__bytes_read.sum"]["value"] * UNIT[s["dram__bytes_read.sum"]["unit"]]
        wr = s["dram__bytes_write.sum"]["value"] * UNIT[s["dram__bytes_write.sum"]["unit"]]
        wf = s["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]["value"]
        inst = s.get("smsp__inst_executed.sum", {}).get("value")
        traffic[f"{cfg}:{M}"] = {"dram_bytes_per_launch": int(rd + wr), "dram_read": int(rd), "dram_write": int(wr),
                                 "smem_wavefronts_per_launch": int(wf),
                                 "warp_instructions_per_launch": int(inst) if inst else None,
                                 "source": os.path.relpath(dst, ROOT) + " (ncu --set full, 1 launch inside bench.py)"}
        print(cfg, M, int(rd + wr), int(wf), s["gpu__time_duration.sum"])
    json.dump(traffic, open(tf, "w"), indent=1)


if __name__ == "__main__":
    main()
