"""Summarise `ncu --set full` reports into the committed profile files.

python tools/ncu_extract.py <round dir> <tag>=<report.ncu-rep> [...]

For each report: writes <round dir>/ncu_full_<tag>_metrics.csv (one row per
profiled kernel, the metrics below) and merges per-kernel entries
"<kernel>@<tag>" into profiles/ncu_summary.json, which bench.py reads for
roofline.traffic (DRAM bytes per launch of the dominant kernel).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "us": 1.0, "ns": 1e-3, "ms": 1e3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def short(name):
    m = re.search(r"(\w+_kernel)<(\d+)>", name) or re.search(r"(\w+_kernel)", name)
    return f"{m.group(1)}<{m.group(2)}>" if m and m.lastindex == 2 else (m.group(1) if m else name[:40])


def main():
    rdir = sys.argv[1]
    os.makedirs(rdir, exist_ok=True)
    sp = os.path.join(ROOT, "profiles", "ncu_summary.json")
    summary = json.load(open(sp)) if os.path.exists(sp) else {"kernels": {}}
    summary["source"] = f"{os.path.relpath(rdir, ROOT)}/ncu_full_*_metrics.csv (ncu --set full --clock-control none)"
    for arg in sys.argv[2:]:
        tag, rep = arg.split("=", 1)
        hdr, units, data = raw(rep)
        ix = {h: i for i, h in enumerate(hdr)}
        cols = [m for m in METRICS if m in ix]
        path = os.path.join(rdir, f"ncu_full_{tag}_metrics.csv")
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["Kernel Name"] + cols)
            w.writerow([""] + [units[ix[c]] for c in cols])
            for r in data:
                w.writerow([r[ix["Kernel Name"]]] + [r[ix[c]] for c in cols])
        for r in data:
            def val(m):
                v = float(r[ix[m]].replace(",", ""))
                return v * SCALE.get(units[ix[m]], 1.0)
            k = short(r[ix["Kernel Name"]]).split("<")[0] + "@" + tag
            rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
            summary["kernels"][k] = {
                "time_us": val("gpu__time_duration.sum"), "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr,
                "dram_pct": val("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                "tensor_pipe_pct": val("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                "tc_pipe_pct": val("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"),
            }
        print(path, len(data), "kernels")
    json.dump(summary, open(sp, "w"), indent=1)


if __name__ == "__main__":
    main()
