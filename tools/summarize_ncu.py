"""Summarise an ncu launch list and a full capture into profiles/.

    python tools/summarize_ncu.py gpurun_out/launches.csv gpurun_out/prof_trace.ncu-rep profiles/r01_c2

Writes <prefix>_launches.txt (per-kernel device time, share of the step;
skipped when the launch list is ""), <prefix>_full.txt (key metrics of the
captured kernel) and profiles/traffic_<config>.json (DRAM bytes per launch,
read by bench.py)."""
import collections
import csv
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        # L1/TEX and L2 (the big-scene kernel is L1/TEX-bound)
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_local_op_ld.sum",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_local_op_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "derived__memory_l2_theoretical_sectors_global_excessive",
        "derived__memory_l1_wavefronts_shared_excessive",
        "l1tex__m_l1tex2xbar_write_sectors_mem_lg_op_st.sum",
        # histogram commits (red) and the path counter (atom)
        "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_red.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum",
        "smsp__inst_executed_op_global_red.sum",
        "lts__t_requests_srcunit_tex_op_red.sum",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        # pipes (round 2: with the 64-byte nodes the ALU pipe, not L1, is the busiest unit)
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__inst_executed_op_local_ld.sum", "smsp__inst_executed_op_local_st.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    d = collections.defaultdict(list)
    for r in rows[h + 1:]:
        try:
            d[r[4]].append(float(r[-1].replace(",", "")))
        except (ValueError, IndexError):
            pass
    return d


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {k: (vals[hdr.index(k)], units[hdr.index(k)]) for k in KEYS if k in hdr}, vals[hdr.index("Kernel Name")]


def main():
    lpath, rep, prefix = sys.argv[1:4]
    config = sys.argv[4] if len(sys.argv) > 4 else "c2"
    d = launches(lpath) if lpath else {}
    tot = sum(sum(v) / len(v) for k, v in d.items() if "ef::" in k)
    lines = ["kernel | launches | mean device time (us) | share of the library's step time",
             "---|---|---|---"]
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
        m = sum(v) / len(v) / 1e3
        share = f"{100 * m * 1e3 / tot:.1f}%" if "ef::" in k else "(torch / bench plumbing)"
        lines.append(f"{k[:70]} | {len(v)} | {m:.1f} | {share}")
    if d:
        open(prefix + "_launches.txt", "w").write(
            "# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised)\n"
            + "\n".join(lines) + "\n")
    m, name = raw(rep)
    body = [f"# ncu --set full --clock-control none, kernel: {name}"]
    for k in KEYS:
        if k in m:
            body.append(f"{k} = {m[k][0]} {m[k][1]}")
    open(prefix + "_full.txt", "w").write("\n".join(body) + "\n")
    rd = float(m["dram__bytes_read.sum"][0].replace(",", ""))
    wr = float(m["dram__bytes_write.sum"][0].replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(m["dram__bytes_read.sum"][1], 1)
    wr *= scale.get(m["dram__bytes_write.sum"][1], 1)
    outdir = os.environ.get("EF_TRAFFIC_DIR", "profiles")   # on the GPU box: a gpurun_out/ subdir
    os.makedirs(outdir, exist_ok=True)
    def pct(k):
        try:
            return float(m[k][0].replace(",", ""))
        except (KeyError, ValueError):
            return None
    util = {"issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
            "l1tex_pct": pct("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_pct": pct("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pipe_pct": pct("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
            "lanes_per_instruction": pct("smsp__thread_inst_executed_per_inst_executed.ratio"),
            "warp_instructions": pct("smsp__inst_executed.sum"),
            "kernel_ms": pct("gpu__time_duration.sum")}
    json.dump({"dram_bytes_per_launch": rd + wr, "read": rd, "write": wr, "source": os.path.basename(rep),
               "utilisation": util,
               "note": f"one ncu --set full capture of {name.split('(')[0]}"},
              open(os.path.join(outdir, f"traffic_{config}.json"), "w"), indent=1)
    print("\n".join(lines))
    print("\n".join(body))


if __name__ == "__main__":
    main()
