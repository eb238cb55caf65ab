"""The C-ABI library loads on a CPU-only host, exports every symbol the
header declares, and its structs match the ctypes mirror byte for byte."""

import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2511_02248_b200 import _native, abi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "opscale_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"OPSC_API\s+[\w\s\*]+?\b(opsc_\w+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _native.load()
    syms = header_symbols()
    assert len(syms) >= 17
    assert set(syms) == set(_native.EXPORTS)
    for s in syms:
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (opsc_\w+)", out))
    assert set(syms) <= exported


def test_library_info_without_gpu():
    L = _native.load()
    assert L.opsc_abi_version() == abi.ABI_VERSION
    assert L.opsc_status_string(abi.ERR_SPACE).decode().startswith("candidate space")
    n = C.c_int(-1)
    L.opsc_device_count(C.cast(C.byref(n), C.c_void_p))
    assert n.value >= 0


SIZES_C = r"""
#include <stdio.h>
#include <stddef.h>
#include "opscale_b200.h"
int main(void) {
  printf("OpscDag %zu %zu %zu %zu\n", sizeof(OpscDag), offsetof(OpscDag, c0), offsetof(OpscDag, out_ptr), offsetof(OpscDag, link_bw));
  printf("OpscGrid %zu %zu %zu\n", sizeof(OpscGrid), offsetof(OpscGrid, menu_off), offsetof(OpscGrid, params_b_max));
  printf("OpscModelSpec %zu %zu\n", sizeof(OpscModelSpec), offsetof(OpscModelSpec, r_cap));
  printf("OpscPlaceSpec %zu %zu\n", sizeof(OpscPlaceSpec), offsetof(OpscPlaceSpec, mem_cap));
  printf("OpscWindows %zu %zu\n", sizeof(OpscWindows), offsetof(OpscWindows, eps));
  printf("OpscDecisions %zu %zu\n", sizeof(OpscDecisions), offsetof(OpscDecisions, devices));
  return 0;
}
"""


def test_struct_layout_matches_ctypes(tmp_path):
    src = tmp_path / "sizes.c"
    src.write_text(SIZES_C)
    exe = tmp_path / "sizes"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    got = {l.split()[0]: [int(x) for x in l.split()[1:]] for l in out.strip().splitlines()}
    exp = {
        "OpscDag": [C.sizeof(abi.OpscDag), abi.OpscDag.c0.offset, abi.OpscDag.out_ptr.offset,
                    abi.OpscDag.link_bw.offset],
        "OpscGrid": [C.sizeof(abi.OpscGrid), abi.OpscGrid.menu_off.offset,
                     abi.OpscGrid.params_b_max.offset],
        "OpscModelSpec": [C.sizeof(abi.OpscModelSpec), abi.OpscModelSpec.r_cap.offset],
        "OpscPlaceSpec": [C.sizeof(abi.OpscPlaceSpec), abi.OpscPlaceSpec.mem_cap.offset],
        "OpscWindows": [C.sizeof(abi.OpscWindows), abi.OpscWindows.eps.offset],
        "OpscDecisions": [C.sizeof(abi.OpscDecisions), abi.OpscDecisions.devices.offset],
    }
    assert got == exp


def test_no_cpu_fallback_on_cpu_host():
    """Without a GPU the planner raises instead of computing on the CPU."""
    if _native.device_count() > 0:
        pytest.skip("GPU present")
    from paper_2511_02248_b200 import DeviceUnavailable, model, planners
    from workloads import scenarios
    dag, prof = scenarios.scenario("cfg1")
    with pytest.raises(DeviceUnavailable):
        planners.brute_force_autoscale(dag, prof, model.WorkloadPoint(10.0, 512, "prefill"),
                                       model.AutoscaleParams(slo=0.5),
                                       model.BruteForceBounds(r_max=2, b_max=1, parallelism=(1,)))
