"""Aggregate an ncu --set full report's warp-stall samples of one kernel by
enclosing device function (dev tool; builds on tools/ncu_stalls.py).

    python tools/ncu_regions.py <report.ncu-rep> <kernel-regex> <cubin-name> [launch-index]
"""
import collections
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import ncu_stalls as N  # noqa: E402

FUNC = re.compile(r"^(?:template <[^>]*>\s*)?(?:static\s+)?(?:__device__|__global__|__host__ __device__)[^(]*?\b(\w+)\(")


def starts(path):
    out = []
    for i, line in enumerate(open(path).read().splitlines()):
        m = FUNC.match(line)
        if m:
            out.append((i + 1, m.group(1)))
    return out


def main():
    report, kernel, cubin = sys.argv[1:4]
    launch = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    hdr, rows = N.sass_page(report, kernel, launch)
    ops = [re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split(" ")[0].split(".")[0] for r in rows if len(r) > 1]
    table = N.pick(N.line_tables(cubin, kernel), ops)
    col = {c: i for i, c in enumerate(hdr)}
    base = int(rows[0][0], 16)
    csrc = os.path.join(N.REPO, "paper_2511_02248_b200", "csrc")
    fstarts = {}
    agg, inst, tot = collections.Counter(), collections.Counter(), 0
    for r in rows:
        if len(r) < len(hdr):
            continue
        f, ln = table.get(int(r[0], 16) - base, ("?", 0))
        if f not in fstarts:
            p = os.path.join(csrc, f)
            fstarts[f] = starts(p) if os.path.exists(p) else []
        name = "?"
        for s, n in fstarts[f]:
            if s <= ln:
                name = n
        key = f"{f}:{name}"
        s = int(r[col["Warp Stall Sampling (All Samples)"]] or 0)
        agg[key] += s
        inst[key] += int(r[col["Instructions Executed"]] or 0)
        tot += s
    for k, v in agg.most_common():
        print(f"{100 * v / max(1, tot):5.1f}%  inst {inst[k]:>8}  {k}")


if __name__ == "__main__":
    main()
