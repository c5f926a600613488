"""Pins for the CPU oracle (runs without a GPU).

The oracle is checked against things other than itself: the paper's printed worked value
(P:1145-1146), closed forms derived from Eq. (2), invariants the paper states (purity Eq. (14),
faithfulness/Clifford invariance/additivity P:105-110), and three mutually independent
evaluations (operator-definition brute force, explicit I/X/Y/Z tensor products, Alg. 2).
"""
import json
import math
import os

import numpy as np
import pytest

import sre_inputs as si

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ALPHAS = [0.5, 1.0, 1.5, 2.0, 3.0]


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_three_modes_agree(oracle_lib, n):
    """brute (operator definition) == pauli (explicit I/X/Y/Z) == fwht (Alg. 2), all alphas."""
    for seed in range(3):
        psi = si.haar(n, 100 + seed)
        b = oracle_lib.sums_brute(psi, ALPHAS)
        p, max_im = oracle_lib.sums_pauli(psi, ALPHAS)
        f = oracle_lib.sums_fwht(psi, ALPHAS)
        assert max_im < 1e-14  # Pauli strings are Hermitian: <P> real
        assert rel(b[:-1], p[:-1]) < 1e-12 and rel(f[:-1], p[:-1]) < 1e-12
        assert abs(b[-1] - p[-1]) < 1e-12 * 4 ** n and abs(f[-1] - p[-1]) < 1e-12 * 4 ** n


@pytest.mark.parametrize("n", [6, 7])
def test_brute_vs_fwht_larger(oracle_lib, n):
    psi = si.brickwall(n, 4, 7 + n)
    b = oracle_lib.sums_brute(psi, [1.0, 2.0, 3.0])
    f = oracle_lib.sums_fwht(psi, [1.0, 2.0, 3.0])
    assert rel(b, f) < 1e-12


def test_pauli_mode_brute_n6(oracle_lib):
    psi = si.haar(6, 9)
    p, mi = oracle_lib.sums_pauli(psi, [2.0])
    f = oracle_lib.sums_fwht(psi, [2.0])
    assert mi < 1e-14 and rel(p[:2], f[:2]) < 1e-12


def test_paper_zero_state_value(oracle_lib):
    """SRE(|0>^16, 2) printed as -0.0 with lost_norm 0.0 (bitwise)."""
    g = json.load(open(os.path.join(GOLD, "paper_zero_state.json")))
    # the full N=16 sweep is a GPU test; the oracle runs the same state at N=12 in full and
    # the paper's N=16 on the two X-strings ranges that carry all the weight and a zero range
    for n in (1, 5, 12):
        m, ln = oracle_lib.sre(si.zero(n), [g["alpha"]], "fwht")
        assert m[0] == 0.0 and math.copysign(1.0, m[0]) == -1.0  # -0.0, as printed
        assert ln == 0.0
    s = oracle_lib.sums_fwht(si.zero(16), [2.0], a_range=(0, 1))
    assert s[0] == 2.0 ** 16 and s[1] == 2.0 ** 16
    s1 = oracle_lib.sums_fwht(si.zero(16), [2.0], a_range=(1, 9))
    assert s1[0] == 0.0 and s1[1] == 0.0


def test_t_state_closed_form(oracle_lib):
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    for a_str, v in g["t_state_N8"].items():
        a = float(a_str)
        assert abs(oracle_lib.t_state_m(a, 8) - v) < 1e-14
    m, ln = oracle_lib.sre(si.t_state(8), [1.0, 2.0, 3.0], "fwht")
    for mi, a in zip(m, [1.0, 2.0, 3.0]):
        assert abs(mi - g["t_state_N8"][str(int(a))]) < 1e-12
    assert abs(ln) < 1e-14
    for n in (1, 2, 3, 4):
        m, _ = oracle_lib.sre(si.t_state(n), [1.0, 2.0, 3.0, 1.5], "brute")
        for mi, a in zip(m, [1.0, 2.0, 3.0, 1.5]):
            assert abs(mi - oracle_lib.t_state_m(a, n)) < 1e-12


def test_product_state_closed_form(oracle_lib):
    for seed in range(4):
        psi, bloch = si.product(6, seed)
        s = oracle_lib.sums_fwht(psi, ALPHAS)
        for i, a in enumerate(ALPHAS):
            assert rel(s[i], oracle_lib.product_state_sums(bloch, a)) < 1e-12


@pytest.mark.parametrize("n", [4, 6, 8])
def test_stabilizer_states_zero(oracle_lib, n):
    """Faithfulness: random Clifford states have M_alpha = 0."""
    for seed in range(3):
        psi = si.random_clifford_state(n, 2 * n, 1000 * n + seed)
        m, ln = oracle_lib.sre(psi, [1.0, 2.0, 3.0, 0.5], "fwht")
        assert max(abs(x) for x in m) < 1e-10
        assert abs(ln) < 1e-12


def test_t_doped_clifford(oracle_lib):
    """Clifford invariance + additivity: M(C(|T>^t|0>^(N-t))) = t M(|T>)."""
    for t in range(0, 5):
        psi = si.t_doped(7, t, 10, 50 + t)
        m, _ = oracle_lib.sre(psi, [2.0, 3.0, 1.0], "fwht")
        for mi, a in zip(m, [2.0, 3.0, 1.0]):
            assert abs(mi - oracle_lib.t_state_m(a, t)) < 1e-10


def test_additivity_and_clifford_invariance(oracle_lib):
    lo, hi = si.haar(4, 5), si.haar(3, 6)
    m_lo, _ = oracle_lib.sre(lo, ALPHAS, "fwht")
    m_hi, _ = oracle_lib.sre(hi, ALPHAS, "fwht")
    m_pair, _ = oracle_lib.sre(np.kron(hi, lo), ALPHAS, "fwht")
    m_scr, _ = oracle_lib.sre(si.scrambled_pair(lo, hi, 8, 3), ALPHAS, "fwht")
    for i in range(len(ALPHAS)):
        assert abs(m_pair[i] - m_lo[i] - m_hi[i]) < 1e-10
        assert abs(m_scr[i] - m_lo[i] - m_hi[i]) < 1e-10


def test_qubit_permutation_invariance(oracle_lib):
    n = 7
    psi = si.haar(n, 77)
    perm = np.random.default_rng(1).permutation(n)
    idx = np.arange(1 << n)
    new = np.zeros_like(idx)
    for j in range(n):
        new |= ((idx >> j) & 1) << perm[j]
    psi2 = np.zeros_like(psi)
    psi2[new] = psi
    s1 = oracle_lib.sums_fwht(psi, ALPHAS)
    s2 = oracle_lib.sums_fwht(psi2, ALPHAS)
    assert rel(s1, s2) < 1e-12


def test_purity_and_parseval_per_x_string(oracle_lib):
    """Eq. (14): sum_P <P>^2 = 2^N; per X-string (Parseval on Eq. (12)):
    sum_b |chi_b(a)|^2 = 2^N sum_x |psi_x|^2 |psi_{x^a}|^2, and chi_0(a) = <psi|X_a|psi>."""
    n = 9
    psi = si.haar(n, 4)
    s, pa = oracle_lib.sums_fwht(psi, [2.0], per_a=True)
    assert abs(s[1] - 2.0 ** n) < 1e-12 * 2 ** n
    idx = np.arange(1 << n)
    p2 = np.abs(psi) ** 2
    for a in (0, 1, 5, 300, 511):
        assert abs(pa[a, 1] - 2 ** n * np.sum(p2 * p2[idx ^ a])) < 1e-13 * 2 ** n
        c = oracle_lib.chi(psi, a)
        assert abs(c[0] - np.vdot(psi, psi[idx ^ a])) < 1e-14
        assert abs(np.sum(np.abs(c) ** 4) - pa[a, 0]) < 1e-12 * max(pa[a, 0], 1.0)


def test_chi_reality(oracle_lib):
    """chi_b(a) is real when a.b is even and imaginary when odd (DESIGN reading C3)."""
    n = 6
    psi = si.haar(n, 11)
    for a in range(0, 64, 7):
        c = oracle_lib.chi(psi, a)
        for b in range(64):
            if bin(a & b).count("1") % 2 == 0:
                assert abs(c[b].imag) < 1e-15
            else:
                assert abs(c[b].real) < 1e-15


def test_range_split_additivity(oracle_lib):
    psi = si.haar(8, 21)
    full = oracle_lib.sums_fwht(psi, ALPHAS)
    parts = sum(oracle_lib.sums_fwht(psi, ALPHAS, a_range=(lo, lo + 64)) for lo in range(0, 256, 64))
    assert rel(full, parts) < 1e-13 or np.max(np.abs(full - parts)) < 1e-10


def test_haar_concentration(oracle_lib):
    """Haar states approach M2 = log2(2^N+3) - 2 (statistical sanity)."""
    n = 10
    vals = [oracle_lib.sre(si.haar(n, 900 + s), [2.0], "fwht")[0][0] for s in range(4)]
    assert abs(np.mean(vals) - oracle_lib.haar_m2(n)) < 40 * 2.0 ** -n * 4


@pytest.mark.parametrize("n", [1, 3, 6])
def test_spectrum_t_state_closed_form(n):
    """Spectrum epilogue pin: |T>^N has t = 2^{-k} with multiplicity C(N,k) 2^k, zeros otherwise."""
    import oracle
    import sre_inputs as si
    np.testing.assert_array_equal(oracle.spectrum(si.t_state(n)), oracle.t_state_spectrum(n))


def test_spectrum_total_and_bins():
    import oracle
    import sre_inputs as si
    c = oracle.spectrum(si.haar(5, 31))
    assert c.sum() == 4 ** 5
    assert c[0] >= 1                       # the identity string: t = 1 -> bin 0
    b = oracle.spectrum_bin(np.array([1.0, 0.75, 0.70, 0.5, 2.0 ** -10, 0.0, 1e-300]))
    assert list(b) == [0, 0, 1, 1, 10, 63, 63]
