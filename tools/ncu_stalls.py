"""Source-line stall breakdown of one kernel from an ncu --set full report
(dev tool, no GPU needed).

ncu's CLI prints per-instruction warp-stall samples only on the SASS source
page; this maps each SASS offset back to its CUDA source line with the line
table of the built library (nvdisasm -g on the kernel's cubin) and aggregates
samples and stall reasons per line.

    python tools/ncu_stalls.py <report.ncu-rep> <kernel-regex> <cubin-name> [launch-index] [top]
    e.g. python tools/ncu_stalls.py gpurun_out/r02_greedy_w1.ncu-rep greedy_kernel k_greedy 1 30
"""

import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_2511_02248_b200", "_lib", "libopscale_b200.so")


def line_tables(cubin, func_re):
    """{function: ({offset: (file, line)}, [opcode, ...])} for the functions
    whose mangled name matches func_re."""
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", f"{cubin}.sm_100a.cubin", LIB], cwd=tmp, check=True,
                   capture_output=True)
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, f"{cubin}.sm_100a.cubin")],
                         check=True, capture_output=True, text=True).stdout
    out, name, cur = {}, None, None
    for ln in txt.splitlines():
        m = re.match(r"//-+ \.text\.(\S+) -+", ln)
        if m:
            name = m.group(1) if re.search(func_re, m.group(1)) else None
            if name:
                out[name] = ({}, [])
            cur = None
            continue
        if not name:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
        if m:
            out[name][0][int(m.group(1), 16)] = cur or ("?", 0)
            out[name][1].append(m.group(2).split(".")[0])
    return out


def pick(tables, page_ops):
    """The instantiation whose opcode sequence is the profiled one."""
    def score(ops):
        n = min(len(ops), len(page_ops))
        return (len(ops) == len(page_ops), sum(a == b for a, b in zip(ops[:n], page_ops[:n])))
    return max(tables.values(), key=lambda t: score(t[1]))[0]


def sass_page(report, kernel, launch):
    out = subprocess.run(["ncu", "-i", report, "--page", "source", "--csv", "--print-source", "sass",
                          "--kernel-id", f"::regex:{kernel}:{launch}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    return rows[hi], rows[hi + 1:]


def main():
    report, kernel, cubin = sys.argv[1:4]
    launch = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 30
    hdr, rows = sass_page(report, kernel, launch)
    page_ops = [re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split(" ")[0].split(".")[0] for r in rows if len(r) > 1]
    table = pick(line_tables(cubin, kernel), page_ops)
    col = {c: i for i, c in enumerate(hdr)}
    stalls = [c for c in hdr if c.startswith("stall_") and "(Not Issued)" not in c]
    base = int(rows[0][0], 16)
    per = collections.defaultdict(lambda: collections.Counter())
    total = collections.Counter()
    for r in rows:
        if len(r) < len(hdr):
            continue
        off = int(r[0], 16) - base
        key = table.get(off, ("?", 0))
        s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        per[key]["samples"] += s
        per[key]["inst"] += int(r[col["Instructions Executed"]] or 0)
        for c in stalls:
            v = int(r[col[c]] or 0)
            per[key][c] += v
            total[c] += v
        total["samples"] += s
    print(f"{kernel} launch {launch}: {total['samples']} samples")
    print("stall reasons: " + ", ".join(f"{c[6:]} {100 * v / max(1, total['samples']):.1f}%"
                                       for c, v in total.most_common() if c != "samples" and v))
    src = {}
    for (f, ln), cnt in sorted(per.items(), key=lambda kv: -kv[1]["samples"])[:top]:
        if f not in src:
            p = os.path.join(REPO, "paper_2511_02248_b200", "csrc", f)
            src[f] = open(p).read().splitlines() if os.path.exists(p) else []
        text = src[f][ln - 1].strip() if 0 < ln <= len(src[f]) else ""
        reasons = ", ".join(f"{c[6:]} {v}" for c, v in cnt.most_common(4) if c.startswith("stall_") and v)
        print(f"{100 * cnt['samples'] / max(1, total['samples']):5.1f}%  {f}:{ln:<5} inst {cnt['inst']:>7}  "
              f"[{reasons}]  {text[:70]}")


if __name__ == "__main__":
    main()
