"""Summarise an ncu report (or a --metrics launch-list CSV) into profiles/.

  python tools/ncu_summary.py gpurun_out/prof_b2.ncu-rep  profiles/r1_k1b.json
  python tools/ncu_summary.py --launches gpurun_out/launches.csv profiles/r1_launches.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "smsp__inst_executed.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected",
]


def from_report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[head.index("Kernel Name")]}
        for k in KEYS:
            if k in head:
                i = head.index(k)
                rec[k] = {"value": r[i], "unit": units[i]}
        out.append(rec)
    return out


def from_launches(path):
    text = open(path).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    total = 0.0
    per = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        name = r["Kernel Name"].split("(")[0]
        per.setdefault(name, [0, 0.0])
        per[name][0] += 1
        per[name][1] += ns
        total += ns
    return {"total_ns": total,
            "kernels": {k: {"launches": c, "ns": t, "share": t / total if total else 0}
                        for k, (c, t) in sorted(per.items(), key=lambda kv: -kv[1][1])}}


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        data = from_launches(sys.argv[2])
        dst = sys.argv[3]
    else:
        data = from_report(sys.argv[1])
        dst = sys.argv[2]
    with open(dst, "w") as f:
        json.dump(data, f, indent=1)
    print(json.dumps(data, indent=1)[:3000])
