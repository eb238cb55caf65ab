"""Device build of the interference exponent's x ** e (opsc_interference_pow,
the code path of the placement kernel): exact for exponents 1, 2, 0.5, the
correctly rounded double otherwise -- so equal to the reference's glibc `**`
wherever glibc rounds correctly (tests/test_pow.py has the host build)."""

import ctypes as C

import numpy as np
import pytest
import torch

from test_pow import correctly_rounded, draws

pytestmark = pytest.mark.gpu


def _device_pow(x, e):
    from paper_2511_02248_b200 import _native
    L = _native.load()
    xt = torch.tensor(x, dtype=torch.float64, device="cuda")
    et = torch.tensor(e, dtype=torch.float64, device="cuda")
    out = torch.empty_like(xt)
    _native.check(L.opsc_interference_pow(xt.data_ptr(), et.data_ptr(), out.data_ptr(), len(x),
                                          torch.cuda.current_stream().cuda_stream), "opsc_interference_pow")
    torch.cuda.synchronize()
    return out.cpu().numpy()


def test_device_pow_correctly_rounded():
    pts = draws(20000, 12)
    got = _device_pow([p[0] for p in pts], [p[1] for p in pts])
    checked = wrong = glibc_diff = glibc_wrong = 0
    for (x, e), g in zip(pts, got.tolist()):
        cr = correctly_rounded(x, e)
        if cr is None:
            continue
        checked += 1
        wrong += g != cr
        glibc_diff += g != x ** e
        glibc_wrong += x ** e != cr
    assert checked > 15000
    assert wrong == 0, wrong
    assert glibc_diff == glibc_wrong and glibc_diff < checked * 0.005, (glibc_diff, glibc_wrong)


def test_device_pow_exact_exponents():
    rng = np.random.default_rng(3)
    x = rng.uniform(1e-6, 2.0, 4096)
    for e, want in ((1.0, x), (2.0, x * x), (0.5, np.sqrt(x))):
        got = _device_pow(x.tolist(), [e] * len(x))
        assert got.tobytes() == want.tobytes(), e
