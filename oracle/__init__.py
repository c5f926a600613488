"""CPU oracle for the exact stabilizer Renyi entropy -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_2601_07824_b200``) never imports it, and the two share no code.

Thin ctypes wrapper around ``sre_oracle.c`` (plain C, long-double arithmetic, OpenMP over
X-strings).  Every function cites the passage of /root/reference/PAPER.md it follows; see the
C file's header.  Also holds the oracle's own finaliser and the closed forms used as pins.

Pinning status: brute, pauli and fwht are pinned against each other
(three independent readings of Eq. (2)), against closed forms (|T>^N, product states,
|0...0>, stabilizer states), against Parseval/purity, and against the paper's printed
|0>^16 console value.  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sre_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile sre_oracle.c into liboracle.so (gcc -O2 -fopenmp). Returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            dp = ctypes.POINTER(ctypes.c_double)
            u64 = ctypes.c_uint64
            lib.oracle_brute.argtypes = [dp, ctypes.c_int, dp, ctypes.c_int, u64, u64, dp, dp]
            lib.oracle_pauli.argtypes = [dp, ctypes.c_int, dp, ctypes.c_int, dp, dp]
            lib.oracle_fwht.argtypes = [dp, ctypes.c_int, dp, ctypes.c_int, u64, u64, dp, dp, dp]
            lib.oracle_finalize.argtypes = [dp, ctypes.c_int, dp, ctypes.c_int, dp, dp]
            lib.oracle_num_threads.argtypes = []
            for f in (lib.oracle_brute, lib.oracle_pauli, lib.oracle_fwht, lib.oracle_finalize,
                      lib.oracle_num_threads):
                f.restype = ctypes.c_int
            _lib = lib
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _prep(psi, alphas):
    psi = np.ascontiguousarray(np.asarray(psi, dtype=np.complex128))
    n = psi.size.bit_length() - 1
    if psi.ndim != 1 or (1 << n) != psi.size:
        raise ValueError("psi must be a 1-D array of length 2^N")
    al = np.ascontiguousarray(np.asarray(list(alphas), dtype=np.float64))
    return psi, n, al


def num_threads() -> int:
    return _load().oracle_num_threads()


def sums_brute(psi, alphas, a_range=None, per_a=False):
    """Eq. (2) by direct operator application, O(8^N). Returns sums[n_alpha+2]."""
    psi, n, al = _prep(psi, alphas)
    lo, hi = a_range if a_range is not None else (0, 1 << n)
    m = al.size + 2
    out = np.zeros(m)
    pa = np.zeros((max(hi - lo, 1), m)) if per_a else None
    rc = _load().oracle_brute(_dp(psi.view(np.float64)), n, _dp(al), al.size, lo, hi, _dp(out),
                              _dp(pa) if per_a else None)
    if rc:
        raise ValueError(f"oracle_brute failed rc={rc}")
    return (out, pa) if per_a else out


def sums_pauli(psi, alphas):
    """Eq. (2) over explicit I/X/Y/Z tensor products. Returns (sums, max|Im<P>|)."""
    psi, n, al = _prep(psi, alphas)
    out = np.zeros(al.size + 2)
    mi = ctypes.c_double(0.0)
    rc = _load().oracle_pauli(_dp(psi.view(np.float64)), n, _dp(al), al.size, _dp(out),
                              ctypes.pointer(mi))
    if rc:
        raise ValueError(f"oracle_pauli failed rc={rc}")
    return out, mi.value


def sums_fwht(psi, alphas, a_range=None, per_a=False):
    """Algorithm 2 literally, complex FWHT per X-string. Returns sums[n_alpha+2]."""
    psi, n, al = _prep(psi, alphas)
    lo, hi = a_range if a_range is not None else (0, 1 << n)
    m = al.size + 2
    out = np.zeros(m)
    pa = np.zeros((max(hi - lo, 1), m)) if per_a else None
    rc = _load().oracle_fwht(_dp(psi.view(np.float64)), n, _dp(al), al.size, lo, hi, _dp(out),
                             _dp(pa) if per_a else None, None)
    if rc:
        raise ValueError(f"oracle_fwht failed rc={rc}")
    return (out, pa) if per_a else out


def chi(psi, a: int) -> np.ndarray:
    """chi_b(a) = <psi|X_a Z_b|psi> for all b via Alg. 2 lines 3-5 (complex, natural b order)."""
    psi, n, al = _prep(psi, [2.0])
    out = np.zeros(al.size + 2)
    c = np.zeros(2 << n)
    rc = _load().oracle_fwht(_dp(psi.view(np.float64)), n, _dp(al), al.size, a, a + 1, _dp(out),
                             None, _dp(c))
    if rc:
        raise ValueError(f"oracle_fwht failed rc={rc}")
    return c.view(np.complex128)


def finalize(sums, n: int, alphas):
    """Eq. (2) from the sums: (list of M_alpha in bits, lost_norm) -- P:99-103."""
    al = np.ascontiguousarray(np.asarray(list(alphas), dtype=np.float64))
    s = np.ascontiguousarray(np.asarray(sums, dtype=np.float64))
    m = np.zeros(al.size)
    ln = ctypes.c_double(0.0)
    _load().oracle_finalize(_dp(s), n, _dp(al), al.size, _dp(m), ctypes.pointer(ln))
    return [float(x) for x in m], ln.value


def sre(psi, alphas, mode: str = "fwht"):
    """(M list, lost_norm) for a state, via the chosen oracle mode."""
    psi = np.asarray(psi, dtype=np.complex128)
    n = psi.size.bit_length() - 1
    if mode == "fwht":
        s = sums_fwht(psi, alphas)
    elif mode == "brute":
        s = sums_brute(psi, alphas)
    elif mode == "pauli":
        s, _ = sums_pauli(psi, alphas)
    else:
        raise ValueError(mode)
    return finalize(s, n, alphas)


# ---------------------------------------------------------------------------------------------
# Closed forms (derived in DESIGN.md "Oracle pins" from the single-qubit expectation values).
# ---------------------------------------------------------------------------------------------
def t_state_m(alpha: float, n: int) -> float:
    """M_alpha(|T>^{(x)N}) in bits: per qubit <I,X,Y,Z> = (1, 1/sqrt2, 1/sqrt2, 0), so
    S_alpha = (1 + 2 * 2^{-alpha})^N and M = N log2((1 + 2^{1-alpha})/2)/(1-alpha); M_1 = N/2."""
    if alpha == 1.0:
        return n / 2.0
    return n * math.log2((1.0 + 2.0 ** (1.0 - alpha)) / 2.0) / (1.0 - alpha)


def product_state_sums(bloch, alpha: float) -> float:
    """S_alpha of a product state with Bloch vectors (x_j, y_j, z_j): prod_j (1 + |x|^{2a} + |y|^{2a} + |z|^{2a})
    (Pauli strings factorise over qubits; additivity P:109)."""
    s = 1.0
    for (x, y, z) in bloch:
        s *= 1.0 + abs(x) ** (2 * alpha) + abs(y) ** (2 * alpha) + abs(z) ** (2 * alpha)
    return s


def haar_m2(n: int) -> float:
    """Haar-average value M_2^Haar = log2(2^N + 3) - 2. Statistical sanity only."""
    return math.log2(2.0 ** n + 3.0) - 2.0


# ---------------------------------------------------------------------------------------------
# Spectrum epilogue (NEXT-2): histogram of t = |<P>|^2 over all 4^N Pauli strings.
# ---------------------------------------------------------------------------------------------
SPECTRUM_BINS = 64


def spectrum_bin(t: np.ndarray) -> np.ndarray:
    """Bin k (0 <= k <= 62) holds round(-log2 t) == k, i.e. t in (2^{-k-1/2}, 2^{-k+1/2}]; bin 63
    holds everything below 2^{-62.5}, exact zeros included.  The decision uses the float64 value's
    exponent and a mantissa-vs-sqrt(2) comparison (DESIGN C22)."""
    t = np.asarray(t, dtype=np.float64)
    m, e = np.frexp(t)                      # t = m 2^e, m in [0.5, 1)
    m2 = 2.0 * m                            # t = m2 2^(e-1), m2 in [1, 2)
    k = -(e - 1) - (m2 > math.sqrt(2.0)).astype(np.int64)   # round(-log2 t)
    k = np.where(t > 0.0, k, SPECTRUM_BINS - 1)
    return np.clip(k, 0, SPECTRUM_BINS - 1)


def spectrum(psi, a_range=None) -> np.ndarray:
    """Counts[64] of t = |chi_b(a)|^2 over b in [0, 2^N) and a in a_range (default all), from the
    oracle's own Alg. 2 chi."""
    psi = np.asarray(psi, dtype=np.complex128)
    n = psi.size.bit_length() - 1
    lo, hi = a_range if a_range is not None else (0, 1 << n)
    counts = np.zeros(SPECTRUM_BINS, dtype=np.int64)
    for a in range(lo, hi):
        c = chi(psi, a)
        t = (c.real ** 2 + c.imag ** 2)
        counts += np.bincount(spectrum_bin(t), minlength=SPECTRUM_BINS)
    return counts


def t_state_spectrum(n: int) -> np.ndarray:
    """|T>^N: per qubit <I,X,Y,Z>^2 = (1, 1/2, 1/2, 0), so t = 2^{-k} with multiplicity
    C(N,k) 2^k (k qubits carrying X or Y, the rest I) and t = 0 otherwise (4^N - 3^N strings)."""
    counts = np.zeros(SPECTRUM_BINS, dtype=np.int64)
    for k in range(n + 1):
        counts[min(k, SPECTRUM_BINS - 1)] += math.comb(n, k) * 2 ** k
    counts[SPECTRUM_BINS - 1] += 4 ** n - 3 ** n
    return counts
