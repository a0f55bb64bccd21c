"""Key counters + top stall reasons of one ncu report.

    python profiles/ncu_brief.py gpurun_out/<tag>.ncu-rep [n_sass_lines]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem"]


def main():
    rep = sys.argv[1]
    nlines = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    print(v[h.index("Kernel Name")][:150])
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print(f"  {k:60s} {v[i]:>16s} {u[i]}")
    st = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v[i])
            except ValueError:
                pass
    print("  stalls/issue:", ", ".join(f"{k} {x:.2f}" for k, x in sorted(st.items(), key=lambda kv: -kv[1])[:8]))
    if nlines:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h = rows[1]
        data = rows[2:]
        i_s = h.index("Warp Stall Sampling (All Samples)")
        i_src = h.index("Source")
        i_ex = h.index("Instructions Executed")
        tot = sum(int(r[i_s]) for r in data) or 1
        for r in sorted(data, key=lambda r: -int(r[i_s]))[:nlines]:
            print(f"  {r[0][-5:]} {int(r[i_s]) / tot:6.1%} {r[i_ex]:>10s}  {r[i_src].strip()[:90]}")


if __name__ == "__main__":
    main()
