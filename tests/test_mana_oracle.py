"""Pins for the qutrit-mana oracle (NEXT-3), independent of the oracle's own arithmetic.

PAPER.md Sec. 2.1 (Eqs. (5)-(10)), Alg. 4/5.  Three evaluations of the same
sums from three readings (phase-space definition, operator form of Alg. 4, Alg. 5) must agree;
closed forms: |0>^N is a stabilizer state (mana 0; P:1401-1403 prints -1.97e-14 at N = 10), the
strange state (|1>-|2>)/sqrt2 has sum_u |W| = 5/3, Wigner normalisation sum_u W = 1,
additivity and Clifford invariance, Cauchy-Schwarz bound sum|W| <= 3^{N/2} for pure states.
"""
import math

import numpy as np
import pytest

from oracle import mana as om
import sre_inputs.qutrit as q


@pytest.mark.parametrize("mode", ["phase_space", "brute", "fwht"])
def test_strange_state(mode):
    s = getattr(om, "sums_" + mode)(q.strange())
    assert s[0] == pytest.approx(5.0, abs=1e-12)           # 3 * sum|W| = 3 * 5/3
    assert s[1] == pytest.approx(3.0, abs=1e-12)
    assert om.mana(q.strange(), mode) == pytest.approx(math.log2(5.0 / 3.0), abs=1e-13)


def test_strange_state_wigner_by_hand():
    """Single-qutrit Wigner function of (|1>-|2>)/sqrt2 by hand: A_0|x> = |-x> swaps |1>,|2>, so
    <A_0> = -1 and W(0) = -1/3; the 8 other points have W = 1/6 each (sum W = 1, sum|W| = 1/3 + 8/6 = 5/3)."""
    s = om.sums_phase_space(q.strange())
    assert s[0] == pytest.approx(3 * (1.0 / 3.0 + 8.0 / 6.0), abs=1e-12)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_three_readings_agree_small(n):
    psi = q.haar(n, 100 + n)
    a = om.sums_phase_space(psi)
    b = om.sums_brute(psi)
    c = om.sums_fwht(psi)
    np.testing.assert_allclose(a, b, rtol=1e-12)
    np.testing.assert_allclose(a, c, rtol=1e-12)


@pytest.mark.parametrize("n", [4, 5])
def test_brute_vs_fwht(n):
    psi = q.brickwall(n, 3, 200 + n)
    np.testing.assert_allclose(om.sums_brute(psi), om.sums_fwht(psi), rtol=1e-12)


@pytest.mark.parametrize("n", [1, 2, 4, 6])
def test_zero_state(n):
    s = om.sums_fwht(q.zero(n))
    assert s[0] == pytest.approx(3.0 ** n, rel=1e-14)
    assert om.mana(q.zero(n)) == pytest.approx(0.0, abs=1e-13)


@pytest.mark.parametrize("n", [2, 4, 6])
def test_wigner_normalisation(n):
    s = om.sums_fwht(q.haar(n, 300 + n))
    assert s[1] == pytest.approx(3.0 ** n, rel=1e-12)
    assert 3.0 ** n <= s[0] <= 3.0 ** n * 3.0 ** (n / 2) + 1e-9   # mana in [0, N/2 log2 3]


def test_additivity():
    a, b = q.haar(2, 7), q.brickwall(3, 2, 8)
    m = om.mana(np.kron(b, a))
    assert m == pytest.approx(om.mana(a) + om.mana(b), abs=1e-12)
    assert om.mana(q.kron([q.strange()] * 4)) == pytest.approx(4 * math.log2(5.0 / 3.0), abs=1e-12)


def test_clifford_invariance():
    rng = np.random.default_rng(11)
    psi = q.haar(5, 12)
    m0 = om.mana(psi)
    m1 = om.mana(q.clifford_circuit(psi, 4, rng))
    assert m1 == pytest.approx(m0, abs=1e-12)
    stab = q.clifford_circuit(q.zero(5), 5, np.random.default_rng(13))
    assert om.mana(stab) == pytest.approx(0.0, abs=1e-12)


def test_range_split():
    psi = q.haar(4, 21)
    whole = om.sums_fwht(psi)
    parts = om.sums_fwht(psi, (0, 30)) + om.sums_fwht(psi, (30, 81))
    np.testing.assert_allclose(whole, parts, rtol=1e-14)
