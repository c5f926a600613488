"""Oracle for pure-state qutrit mana (NEXT-3) -- TEST INFRASTRUCTURE ONLY.

Wraps three evaluations in ``sre_oracle.c`` of the same two sums over the 9^N phase-space
points u = (a, b) of N qutrits (Sec. 2.1, Eqs. (4)-(10); Sec. 3.3,
Alg. 4/5):

  sums[0] = sum_u |<psi|A_u|psi>|   -> mana = log2(sums[0] / 3^N)        (Eq. (10), reading C18)
  sums[1] = sum_u  <psi|A_u|psi>    -> 3^N for every normalised state     (sum_u W(u) = 1)

  sums_phase_space : Eqs. (5)-(7) literally: dense T_u, A_0 = 3^{-N} sum_u T_u, A_u = T_u A_0 T_u^+ (N <= 3)
  sums_brute       : Alg. 4 semantics, A_ab = D A_0 D^+ with A_0|x> = |-x> applied as operators (N <= 5)
  sums_fwht        : Alg. 5 literally, per X-string a: v_x = conj(psi_{x-a}) psi_{-x-a}, F_3^{(x)N}, sum |chi|

Index convention: x = sum_j x_j 3^j (qutrit j is ternary digit j).
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _dp, _load

_ready = False


def _lib():
    global _ready
    lib = _load()
    if not _ready:
        dp = ctypes.POINTER(ctypes.c_double)
        u64 = ctypes.c_uint64
        lib.oracle_mana_brute.argtypes = [dp, ctypes.c_int, dp]
        lib.oracle_mana_phase_space.argtypes = [dp, ctypes.c_int, dp]
        lib.oracle_mana_fwht.argtypes = [dp, ctypes.c_int, u64, u64, dp]
        for f in (lib.oracle_mana_brute, lib.oracle_mana_phase_space, lib.oracle_mana_fwht):
            f.restype = ctypes.c_int
        _ready = True
    return lib


def n_qutrits(size: int) -> int:
    n, d = 0, 1
    while d < size:
        d *= 3
        n += 1
    if d != size:
        raise ValueError("psi must have length 3^N")
    return n


def _prep(psi):
    psi = np.ascontiguousarray(np.asarray(psi, dtype=np.complex128))
    if psi.ndim != 1:
        raise ValueError("psi must be 1-D")
    return psi, n_qutrits(psi.size)


def sums_phase_space(psi) -> np.ndarray:
    psi, n = _prep(psi)
    out = np.zeros(2)
    if _lib().oracle_mana_phase_space(_dp(psi.view(np.float64)), n, _dp(out)):
        raise ValueError("oracle_mana_phase_space: N must be 1..3")
    return out


def sums_brute(psi) -> np.ndarray:
    psi, n = _prep(psi)
    out = np.zeros(2)
    if _lib().oracle_mana_brute(_dp(psi.view(np.float64)), n, _dp(out)):
        raise ValueError("oracle_mana_brute: N must be 1..6")
    return out


def sums_fwht(psi, a_range=None) -> np.ndarray:
    psi, n = _prep(psi)
    lo, hi = a_range if a_range is not None else (0, 3 ** n)
    out = np.zeros(2)
    if _lib().oracle_mana_fwht(_dp(psi.view(np.float64)), n, lo, hi, _dp(out)):
        raise ValueError("oracle_mana_fwht: bad N or a-range")
    return out


def mana(psi, mode: str = "fwht") -> float:
    """log2(sum_u |W(u)|) with W(u) = <psi|A_u|psi>/3^N (Eqs. (8)-(10))."""
    psi, n = _prep(psi)
    s = {"fwht": sums_fwht, "brute": sums_brute, "phase_space": sums_phase_space}[mode](psi)
    return math.log2(s[0] / 3.0 ** n)


def strange_mana() -> float:
    """Closed form for the strange state (|1> - |2>)/sqrt2: W = (1/3)(...) gives sum|W| = 5/3."""
    return math.log2(5.0 / 3.0)


# ---------------------------------------------------------------------------------------------
# Mixed states (NEXT-4): rho as a 3^N x 3^N array; passed to C column-major (Alg. 6's input).
# ---------------------------------------------------------------------------------------------
def _rho_prep(rho):
    rho = np.asarray(rho, dtype=np.complex128)
    if rho.ndim != 2 or rho.shape[0] != rho.shape[1]:
        raise ValueError("rho must be a square 2-D array")
    n = n_qutrits(rho.shape[0])
    flat = np.ascontiguousarray(rho.flatten(order="F"))     # flat[r + c 3^N] = rho[r, c]
    return flat, n


def _mixed_lib():
    lib = _lib()
    dp = ctypes.POINTER(ctypes.c_double)
    for f in (lib.oracle_mana_mixed_phase_space, lib.oracle_mana_mixed_alg6):
        f.argtypes = [dp, ctypes.c_int, dp]
        f.restype = ctypes.c_int
    return lib


def sums_mixed_phase_space(rho) -> np.ndarray:
    """sum_u |Tr(rho A_u)|, sum_u Tr(rho A_u) from the definition (Eqs. (5)-(9)); N <= 4."""
    flat, n = _rho_prep(rho)
    out = np.zeros(2)
    if _mixed_lib().oracle_mana_mixed_phase_space(_dp(flat.view(np.float64)), n, _dp(out)):
        raise ValueError("oracle_mana_mixed_phase_space: N must be 1..4")
    return out


def sums_mixed_alg6(rho) -> np.ndarray:
    """Alg. 6 literally (Vec_N + leg sweep with the dense 9x9 M); N <= 8."""
    flat, n = _rho_prep(rho)
    out = np.zeros(2)
    if _mixed_lib().oracle_mana_mixed_alg6(_dp(flat.view(np.float64)), n, _dp(out)):
        raise ValueError("oracle_mana_mixed_alg6: N must be 1..8")
    return out


def mana_mixed(rho, mode: str = "alg6") -> float:
    rho = np.asarray(rho)
    n = n_qutrits(rho.shape[0])
    s = {"alg6": sums_mixed_alg6, "phase_space": sums_mixed_phase_space}[mode](rho)
    return math.log2(s[0] / 3.0 ** n)


def mixed_strange_mana(p: float) -> float:
    """rho = p |S><S| + (1-p) I/3 (S the strange state): W(0) = (1-4p)/9, the other 8 points
    (2+p)/18 each, so sum|W| = (7+8p)/9 for p >= 1/4 and 1 below."""
    return math.log2(max(1.0, (7.0 + 8.0 * p) / 9.0))
