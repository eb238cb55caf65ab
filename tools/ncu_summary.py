"""Summarise ncu outputs brought back from gpurun into profiles/.

    python tools/ncu_summary.py launches <launches.csv> <out.md>
    python tools/ncu_summary.py full <report.ncu-rep> <out.json> [kernel-regex]

`launches` groups the per-launch gpu__time_duration of a bench run (cold
cache, serialised under ncu: compare SHARES, not absolutes). `full` extracts
the metrics the roofline and the judge cite from one `--set full` capture.
"""

import csv
import io
import json
import re
import subprocess
import sys
from collections import OrderedDict


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    n = 0
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).strip()
        v = float(r[vi].replace(",", ""))
        unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
        scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                 "msecond": 1.0}.get(unit, 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
        n += 1
    total = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.3f} | {t / total:.1%} |")
    lines.append(f"\n{n} launches, {total:.3f} ms total (ncu-serialised, cold cache).")
    # the bench step's own kernels: everything but the live FP64-peak
    # microbenchmark (a measurement helper) and torch fill kernels (L2 flush,
    # buffer resets outside the timed region)
    step = {k: v for k, v in agg.items() if k.startswith(("opsc::", "void opsc::")) and "peak" not in k}
    st = sum(v[1] for v in step.values())
    if st > 0:
        lines.append("\nShare of the planning step (opsc kernels only):\n")
        lines.append("| kernel | share of step |")
        lines.append("|---|---|")
        for k, (c, t) in sorted(step.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {t / st:.2%} |")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    "gpu__time_duration.sum", "sm__cycles_active.avg", "smsp__cycles_active.avg",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warp_latency_per_inst_issued.ratio",
    "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_inst_executed_op_shared_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
]


def full(path, out, regex=None):
    cmd = ["ncu", "-i", path, "--page", "raw", "--csv"]
    txt = subprocess.run(cmd, capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        rec = dict(zip(hdr, r))
        name = rec.get("Kernel Name", "")
        if regex and not re.search(regex, name):
            continue
        m = {}
        for k in WANT:
            if k in rec:
                u = units[hdr.index(k)]
                try:
                    m[k] = [float(rec[k].replace(",", "")), u]
                except ValueError:
                    m[k] = [rec[k], u]
        res.append({"kernel": name, "metrics": m})
    summary = {"report": path, "kernels": res}
    if res:
        m = res[0]["metrics"]
        rd = m.get("dram__bytes_read.sum", [0, "byte"])
        wr = m.get("dram__bytes_write.sum", [0, "byte"])
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        summary["dram_bytes_per_launch"] = rd[0] * scale.get(rd[1], 1) + wr[0] * scale.get(wr[1], 1)
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
