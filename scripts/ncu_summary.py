"""Summarise an ncu report (run here, no GPU): key throughput / stall metrics."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard", "lts__t_bytes.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")][:90]
        print("kernel:", name)
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:60s} {r[i]:>16s} {units[i]}")
        stalls = [(h[i], r[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled_") and not h[i].endswith("not_issued")]
        tot = sum(float(v or 0) for _, v in stalls) or 1
        top = sorted(stalls, key=lambda kv: -float(kv[1] or 0))[:8]
        print("  top stall reasons (pc sampling):", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')}={float(v)/tot*100:.0f}%" for k, v in top))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
