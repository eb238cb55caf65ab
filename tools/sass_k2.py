"""Dump the SASS of K2's hottest basic block (dev tool, no GPU needed).

For each compose_kernel instantiation named on the command line (template
args NJ,MODE,KREG), cuobjdump the built library, split the function into
basic blocks at branch targets, and print the block with the most DADD
instructions plus an opcode histogram of it: the per-candidate inner loop
(DADD = path extension, DSETP = SLO compare, SEL = feasible-prefix count).

    python tools/sass_k2.py 24,2,0 6,2,1 > profiles/r02_k2_sass.txt
"""
import collections
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "paper_2511_02248_b200", "_lib", "libopscale_b200.so")


def functions(text):
    out, name, body = {}, None, []
    for line in text.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                out[name] = body
            name, body = m.group(1), []
        elif name:
            body.append(line)
    if name:
        out[name] = body
    return out


def blocks(body):
    ins = []
    for line in body:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    targets = set()
    for _, t in ins:
        m = re.search(r"BRA\s.*?`?\(\.L_x_\d+\)|BRA\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", t)
        if m and m.group(1):
            targets.add(int(m.group(1), 16))
    cur, res = [], []
    for addr, t in ins:
        if addr in targets and cur:
            res.append(cur)
            cur = []
        cur.append((addr, t))
        if t.split()[0].lstrip("@!UP0123456789T,").startswith(("BRA", "EXIT", "RET")) or " BRA " in f" {t} ":
            res.append(cur)
            cur = []
    if cur:
        res.append(cur)
    return res


def opcode(t):
    t = re.sub(r"^@!?U?P[T0-9]+\s+", "", t)
    return t.split()[0].split(".")[0]


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    fns = functions(sass)
    for arg in sys.argv[1:]:
        nj, mode, kreg = arg.split(",")
        want = f"compose_kernelILi{nj}ELi{mode}ELb{kreg}E"
        name = next(n for n in fns if want in n)
        bl = max(blocks(fns[name]), key=lambda b: sum(opcode(t) == "DADD" for _, t in b))
        hist = collections.Counter(opcode(t) for _, t in bl)
        print(f"== compose_kernel<{nj},{mode},{int(kreg)}>  ({name})")
        print(f"hottest block: {len(bl)} instructions at 0x{bl[0][0]:04x}; opcode histogram: "
              + ", ".join(f"{k} {v}" for k, v in hist.most_common()))
        for addr, t in bl:
            print(f"  /*{addr:04x}*/ {t}")
        print()


if __name__ == "__main__":
    main()
