"""Summarise an ncu --set full report: key throughput counters, stall mix and
the top stalled SASS lines.  Usage: python tools/ncu_summary.py rep.ncu-rep [kernel-regex]"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__shared_mem_per_block_dynamic", "lts__t_bytes.sum",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    h, units, vals = raw(rep)
    res = []
    for v in vals:
        d = {"kernel": v[h.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in h:
                d[k] = v[h.index(k)] + " " + units[h.index(k)]
        st = {h[i].replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[i])
              for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h[i].endswith("not_issued") and v[i].replace(".", "").isdigit()}
        tot = sum(st.values()) or 1
        d["stalls_pct"] = {k: round(100 * x / tot, 1) for k, x in sorted(st.items(), key=lambda t: -t[1])[:8]}
        res.append(d)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
