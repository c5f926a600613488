"""Pins for the mixed-state mana oracle (NEXT-4): Alg. 6 against the phase-space
definition W_u = Tr(rho A_u)/3^N (Eqs. (5)-(9)), against the pure-state Alg. 5 oracle for
rho = |psi><psi|, and against closed forms: p|S><S| + (1-p) I/3 (strange-state mixture),
I/3^N (W = 9^-N everywhere), Tr rho normalisation, additivity, stabilizer mixtures."""
import math

import numpy as np
import pytest

from oracle import mana as om
import sre_inputs.qutrit as q


@pytest.mark.parametrize("p", [1.0, 0.8, 0.5, 0.3, 0.25, 0.1, 0.0])
def test_strange_mixture_closed_form(p):
    rho = q.mixed_strange(p)
    for mode in ("alg6", "phase_space"):
        assert om.mana_mixed(rho, mode) == pytest.approx(om.mixed_strange_mana(p), abs=1e-13)


@pytest.mark.parametrize("n", [1, 2, 3])
def test_alg6_vs_definition(n):
    rho = q.random_mixed(n, 3, 40 + n)
    np.testing.assert_allclose(om.sums_mixed_alg6(rho), om.sums_mixed_phase_space(rho), rtol=1e-12)


@pytest.mark.parametrize("n", [1, 3, 5])
def test_pure_state_reduces_to_alg5(n):
    psi = q.brickwall(n, 3, 50 + n) if n > 1 else q.haar(1, 50)
    np.testing.assert_allclose(om.sums_mixed_alg6(q.density(psi)), om.sums_fwht(psi), rtol=1e-12)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_maximally_mixed(n):
    s = om.sums_mixed_alg6(np.eye(3 ** n) / 3 ** n)
    assert s[0] == pytest.approx(3.0 ** n, rel=1e-13) and s[1] == pytest.approx(3.0 ** n, rel=1e-13)


def test_trace_normalisation_and_additivity():
    a, b = q.random_mixed(2, 2, 61), q.random_mixed(2, 5, 62)
    sa, sb = om.sums_mixed_alg6(a), om.sums_mixed_alg6(b)
    assert sa[1] == pytest.approx(9.0, rel=1e-13)
    # qutrits 0..1 from a, 2..3 from b: index x = x_a + 9 x_b  <->  kron(b, a)
    assert om.mana_mixed(np.kron(b, a)) == pytest.approx(om.mana_mixed(a) + om.mana_mixed(b), abs=1e-12)


def test_stabilizer_mixture_and_reduced_state():
    rng = np.random.default_rng(71)
    s1 = q.clifford_circuit(q.zero(3), 4, rng)
    s2 = q.clifford_circuit(q.zero(3), 4, rng)
    rho = 0.3 * q.density(s1) + 0.7 * q.density(s2)
    assert om.mana_mixed(rho) == pytest.approx(0.0, abs=1e-12)      # convex hull of stabilizers
    psi = q.brickwall(5, 3, 72)
    red = q.reduced(psi, 3)
    assert np.trace(red).real == pytest.approx(1.0, abs=1e-13)
    assert 0.0 <= om.mana_mixed(red) <= om.mana(psi) + 1e-12        # monotone under partial trace
