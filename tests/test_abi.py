"""The C ABI without a GPU: the library loads, exports every entry point include/sre.h declares,
validates arguments before touching a device, and its host-side finaliser matches the oracle's."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2601_07824_b200 import _build
    _build.build()
    import paper_2601_07824_b200 as sre
    return sre.load()


def test_exports_every_declared_symbol(lib):
    hdr = open(os.path.join(ROOT, "include", "sre.h")).read()
    names = set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(sre_[a-z_0-9]+)\(", hdr, re.M))
    assert {"sre_exact", "sre_exact_batched", "sre_partial_sums", "sre_finalize", "sre_workspace_size",
            "sre_chi", "sre_norm2", "sre_status_string", "sre_last_error"} <= names
    for n in names:
        assert hasattr(lib, n), n


def test_library_is_sm100a_only():
    import subprocess
    so = os.path.join(ROOT, "paper_2601_07824_b200", "libsre_b200.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_validation_before_device(lib):
    import paper_2601_07824_b200 as sre
    dp = ctypes.POINTER(ctypes.c_double)
    al = np.array([2.0])
    out = np.zeros(1)
    buf = np.zeros(16, dtype=np.complex128)
    p = ctypes.c_void_p(buf.ctypes.data)
    a = al.ctypes.data_as(dp)
    o = out.ctypes.data_as(dp)
    assert lib.sre_exact(None, 4, a, 1, o, None) == 1                     # NULL psi
    assert lib.sre_exact(p, 0, a, 1, o, None) == 2                        # N out of range
    assert lib.sre_exact(p, 27, a, 1, o, None) == 2
    bad = np.array([-1.0]).ctypes.data_as(dp)
    assert lib.sre_exact(p, 4, bad, 1, o, None) == 1                      # alpha <= 0
    assert lib.sre_exact(p, 4, a, 0, o, None) == 1                        # n_alpha = 0
    assert lib.sre_exact(p, 4, a, 17, o, None) == 1                       # n_alpha > 16
    assert lib.sre_partial_sums(p, 4, 1, 5, 3, a, 1, p, 1 << 20, p, None) == 2   # a_begin > a_end
    assert lib.sre_partial_sums(p, 4, 1, 0, 17, a, 1, p, 1 << 20, p, None) == 2  # a_end > 2^N
    assert out[0] == 0.0                                                  # untouched on error
    assert sre.workspace_size(20, 1, 1) > 8 * (1 << 20) * 8
    assert lib.sre_workspace_size(0, 1, 1) == 0
    assert lib.sre_status_string(3) == b"state not normalised"


def test_finalize_matches_oracle(lib, oracle_lib):
    import paper_2601_07824_b200 as sre
    import sre_inputs as si
    alphas = [0.5, 1.0, 2.0, 3.0]
    for n in (3, 6):
        s = oracle_lib.sums_fwht(si.haar(n, 5), alphas)
        m_lib, ln_lib = sre.finalize(s, n, alphas)
        m_or, ln_or = oracle_lib.finalize(s, n, alphas)
        assert np.max(np.abs(m_lib[0] - np.array(m_or))) < 1e-14
        assert abs(ln_lib[0] - ln_or) < 1e-16
    m, ln = sre.finalize(np.array([2.0 ** 16, 2.0 ** 16, 0.0]), 16, [2.0])
    assert m[0, 0] == 0.0 and math.copysign(1.0, m[0, 0]) == -1.0 and ln[0] == 0.0


def test_mana_finalize_host(lib):
    """sre_mana_finalize (host-side Eq. (10), no GPU): mana = log2(S_abs / 3^N), ||psi||^2 = S_sum / 3^N;
    the strange state's sum |W| = 5/3 per qutrit (DESIGN section 15 pins) gives N log2(5/3)."""
    from paper_2601_07824_b200 import SreError, qutrit
    for n in (1, 4, 12):
        m, n2 = qutrit.finalize([3.0 ** n * (5.0 / 3.0) ** n, 3.0 ** n], n)
        assert abs(m - n * math.log2(5.0 / 3.0)) < 1e-13 and abs(n2 - 1.0) < 1e-15
    m, n2 = qutrit.finalize(np.array([3.0 ** 10, 3.0 ** 10 * 0.5]), 10)   # stabilizer: mana 0
    assert m == 0.0 and n2 == 0.5
    for bad in (([0.0, 1.0], 3), ([1.0, 1.0], 0), ([1.0, 1.0], 17)):
        with pytest.raises(SreError):
            qutrit.finalize(*bad)
