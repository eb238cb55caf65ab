"""Build libopscale_b200.so in-tree for sm_100a (nvcc, static cudart).

    python -m paper_2511_02248_b200.build [--verbose]

Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo (ncu source
view), --fmad=false (no DFMA contraction: the bit-exactness contract of
SURVEY.md Appendix A). The .so lands in paper_2511_02248_b200/_lib/, which
is git-ignored but travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT, "libopscale_b200.so")
SOURCES = ["k_menu.cu", "k_compose.cu", "k_model.cu", "k_materialize.cu", "k_greedy.cu", "k_windowize.cu", "k_peer.cu",
           "k_place.cu",
           "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
] + os.environ.get("OPSC_NVCC_EXTRA", "").split()


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False):
    os.makedirs(OUT, exist_ok=True)
    header = os.path.join(os.path.dirname(HERE), "include", "opscale_b200.h")
    common = [os.path.join(CSRC, h) for h in sorted(os.listdir(CSRC)) if h.endswith(".cuh")] + [header]
    objs = []
    log = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + common):
            cmd = [NVCC, *FLAGS, "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            log.append(r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if force or _stale(LIB, objs):
        cmd = [NVCC, "-shared", "-cudart", "static", "-gencode", "arch=compute_100a,code=sm_100a",
               "-o", LIB, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    with open(os.path.join(OUT, "ptxas.log"), "w") as fh:  # this build's compiles only
        fh.write("".join(log))
    if verbose:
        print("".join(log))
    return LIB


if __name__ == "__main__":
    print(build(verbose="--verbose" in sys.argv, force="--force" in sys.argv))
