"""Pins for the thermodynamic-integration oracle (NEXT-1, Sec. 3.2.2-3.2.4) on CPU."""
import math

import numpy as np
import pytest

import sre_inputs as si


@pytest.fixture(scope="module")
def mco(oracle_lib):
    import oracle.mc as m
    return m


def test_simpson_weights(mco):
    for L in (3, 5, 21):
        b, w = mco.simpson(L)
        assert abs(sum(w) - 1.0) < 1e-15
        for p in range(4):                       # exact for cubics
            assert abs(sum(wi * bi ** p for bi, wi in zip(b, w)) - 1.0 / (p + 1)) < 1e-14
    with pytest.raises(ValueError):
        mco.simpson(4)                           # even L: reading C17


def test_t_state_energies_closed_form(mco):
    """|T>^N: S(a) = 2^{-|a|} so f(a) = |a| ln 2 (natural log, reading C15), and
    <f>_beta = N ln 2 / (2^beta + 1); int_0^1 = N ln2 (2 - log2 3) => M_2 = N log2(4/3) with the
    + sign of reading C16 (Alg. 3's printed sign would give -M_2)."""
    n = 4
    f = mco.all_energies(si.t_state(n))
    a = np.arange(1 << n)
    pop = np.array([bin(x).count("1") for x in a])
    assert np.max(np.abs(f - pop * math.log(2.0))) < 1e-12
    for beta in (0.0, 0.3, 1.0):
        assert abs(mco.mean_f_exact(f, beta) - n * math.log(2.0) / (2.0 ** beta + 1.0)) < 1e-12
    m = mco.ti_exact(si.t_state(n), 101)
    assert abs(m - n * math.log2(4.0 / 3.0)) < 1e-7


def test_ti_converges_to_exact_sre(oracle_lib, mco):
    psi = si.haar(6, 31)
    exact = oracle_lib.sre(psi, [2.0])[0][0]
    errs = [abs(mco.ti_exact(psi, L) - exact) for L in (5, 11, 41)]
    assert errs[2] < 1e-6 and errs[2] < errs[0]


def test_ti_regularised_converges_to_exact_sre(oracle_lib, mco):
    """eps > 0: M_2 = -log2(e^{-I} - eps) removes the regulariser exactly, so the quadrature
    still converges to the unregularised M_2 (a plain I / ln 2 would be biased by ~eps 2^N / S_2)."""
    psi = si.haar(6, 31)
    exact = oracle_lib.sre(psi, [2.0])[0][0]
    for eps in (1e-3, 1e-2):
        assert abs(mco.ti_exact(psi, 41, eps) - exact) < 1e-6
        biased = sum(w * mco.mean_f_exact(mco.all_energies(psi, eps), b)
                     for b, w in zip(*mco.simpson(41))) / math.log(2.0)
        assert abs(biased - exact) > 1e-3


def test_replay_chain_samples_boltzmann(mco):
    """Detailed-balance check at desk scale: a long beta = 1 chain's pattern frequencies follow
    Pi_1(a) = S(a)/S_2 (Eq. (18)) within multinomial error."""
    n = 3
    psi = si.haar(n, 5)
    f = mco.all_energies(psi)
    pi = np.exp(-f) / np.exp(-f).sum()
    L, steps = 3, 20000
    streams = si.mc_streams(11, L, steps, n)
    # replay only the beta = 1 chain (index L-1) and histogram its patterns
    init, flips, uni = streams
    a, fa = int(init[-1]), f[int(init[-1])]
    counts = np.zeros(1 << n)
    for s in range(steps):
        p = a ^ (1 << int(flips[s, -1, 0]))
        if uni[s, -1] < min(1.0, math.exp(-(f[p] - fa))):
            a, fa = p, f[p]
        counts[a] += 1
    emp = counts / steps
    assert np.max(np.abs(emp - pi) / np.sqrt(pi * (1 - pi) / steps * 30)) < 5.0  # tau ~ a few steps


def test_mc_replay_close_to_ti(mco):
    n, L = 5, 5
    psi = si.haar(n, 8)
    streams = si.mc_streams(3, L, 4050, n)
    means, acc, _ = mco.mc_replay(psi, L, streams, 50, 4000)
    b, w = mco.simpson(L)
    m_mc = float(np.dot(w, means)) / math.log(2.0)
    m_ti = mco.ti_exact(psi, L)
    assert abs(m_mc - m_ti) < 0.05
    assert acc[0] == 4000                        # beta = 0: every proposal accepted
