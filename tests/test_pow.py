"""The interference exponent's x ** e (paper_2511_02248_b200/csrc/opsc_pow.cuh).

The reference computes `excess ** params.exponent` (perfmodel.py:187) with
glibc's pow. The placement kernel evaluates exp(e log x) in double-double and
rounds once; here the same header is compiled as plain C++ with g++ and every
result is compared with a 60-digit decimal evaluation (must be the correctly
rounded double) and with Python's `**` (glibc: equal except where glibc
itself misrounds). The device build of the same code is checked in
tests/test_gpu_pow.py."""

import math
import os
import random
import shutil
import subprocess
from decimal import Decimal, getcontext

import pytest

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2511_02248_b200", "csrc")

DRIVER = r"""
#include <cstdio>
#include "opsc_pow.cuh"
int main() {
  double x, e;
  while (scanf("%la %la", &x, &e) == 2) printf("%a\n", opsc_pow::pow_rn(x, e));
}
"""


def draws(n, seed):
    """(excess, exponent) pairs: the placement's range (excess in (0, 2],
    exponent in [0.5, 2]) plus wider magnitudes and negative exponents."""
    rnd = random.Random(seed)
    out = []
    for i in range(n):
        k = i % 4
        x = (rnd.uniform(1e-9, 2.0) if k == 0 else rnd.uniform(0, 1) ** 3 if k == 1
             else rnd.uniform(0.5, 50.0) if k == 2 else math.ldexp(rnd.uniform(0.5, 1.0), rnd.randint(-900, 900)))
        e = rnd.uniform(0.5, 2.0) if i % 5 else rnd.uniform(-3.0, 3.0)
        if x > 0:
            out.append((x, e))
    return out


def correctly_rounded(x, e):
    """pow(x, e) rounded to nearest from a 60-digit evaluation; None when
    |e log x| > 708 (the kernel hands those to the library pow)."""
    getcontext().prec = 60
    z = Decimal(e) * Decimal(x).ln()
    if abs(z) > 708:
        return None
    return float(z.exp())


@pytest.fixture(scope="module")
def host_pow(tmp_path_factory):
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("g++ not available")
    d = tmp_path_factory.mktemp("pow")
    src, exe = d / "drv.cpp", d / "drv"
    src.write_text(DRIVER)
    subprocess.run([cxx, "-O2", "-ffp-contract=off", "-I", HDR, str(src), "-o", str(exe)], check=True)

    def run(pts):
        inp = "".join(f"{x.hex()} {e.hex()}\n" for x, e in pts)
        out = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True).stdout.split()
        return [float.fromhex(s) for s in out]
    return run


def test_pow_rn_is_correctly_rounded(host_pow):
    pts = draws(20000, 11)
    got = host_pow(pts)
    checked = wrong = glibc_diff = glibc_wrong = 0
    for (x, e), g in zip(pts, got):
        cr = correctly_rounded(x, e)
        if cr is None:
            continue
        checked += 1
        wrong += g != cr
        ge = x ** e
        glibc_diff += g != ge
        glibc_wrong += ge != cr
    assert checked > 15000
    assert wrong == 0, wrong
    # every disagreement with glibc is one of glibc's own misroundings (~0.1%)
    assert glibc_diff == glibc_wrong and glibc_diff < checked * 0.005, (glibc_diff, glibc_wrong)


def test_pow_rn_special_values(host_pow):
    pts = [(1.0, 1.7), (2.0, 0.0), (0.25, 1.5), (4.0, 1.5), (9.0, 0.5), (2.0, 10.0), (1e-310, 1.5),
           (1e300, 3.0), (1e-300, 3.0), (0.5, -2.0), (math.inf, 1.5), (0.0, 1.5)]
    got = host_pow(pts)
    for (x, e), g in zip(pts, got):
        assert g == (math.pow(x, e) if x < 1e300 else math.inf), (x, e, g)
