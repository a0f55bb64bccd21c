"""Summarise ncu reports / launch lists into profiles/<tag>_summary.json.

    python profiles/summarize.py r01 gpurun_out
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def raw(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")]}
    stalls = {}
    for i, k in enumerate(h):
        if k in KEYS:
            try:
                val = float(v[i].replace(",", ""))
            except ValueError:
                continue
            res[k] = val * UNIT.get(u[i], 1) if u[i] in UNIT else val
            if u[i] in UNIT:
                res[k + ".unit"] = "bytes" if "byte" in u[i] else "s"
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
            try:
                stalls[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = int(float(v[i]))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1
    res["stall_share_top"] = {k: round(c / tot, 3) for k, c in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
    rd, wr = res.get("dram__bytes_read.sum"), res.get("dram__bytes_write.sum")
    if rd is not None and wr is not None:
        res["dram_bytes_total"] = rd + wr
    return res


def launches(path: Path) -> list:
    text = path.read_text()
    lines = [l for l in text.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    h = rows[0]
    out = []
    for r in rows[1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append({"kernel": d["Kernel Name"].split("(")[0][:120], "ns": float(d["Metric Value"].replace(",", ""))})
    return out


def main():
    tag, src = sys.argv[1], Path(sys.argv[2])
    summary = {"tag": tag, "reports": {}}
    for rep in sorted(src.glob(f"{tag}_*.ncu-rep")):
        summary["reports"][rep.stem] = raw(rep)
    lp = src / f"{tag}_launches.csv"
    if lp.exists():
        ls = launches(lp)
        total = sum(x["ns"] for x in ls) or 1
        by = {}
        for x in ls:
            by.setdefault(x["kernel"], []).append(x["ns"])
        summary["launch_list"] = {k: {"launches": len(v), "mean_ns": sum(v) / len(v), "share": sum(v) / total}
                                  for k, v in by.items()}
    out = Path(__file__).resolve().parent / f"{tag}_summary.json"
    out.write_text(json.dumps(summary, indent=1))
    print(out)


if __name__ == "__main__":
    main()
