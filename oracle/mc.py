"""Oracle for the thermodynamic-integration sampler (NEXT-1) -- TEST INFRASTRUCTURE ONLY.

Plain Python written from PAPER.md Sec. 3.2.2-3.2.4 with the readings of
DESIGN.md C15-C17 (natural log in f, M_2 = +(1/ln 2) sum_l w_l <f>_l, odd L with Simpson weights).
Shares no code with paper_2601_07824_b200/mc.py; energies come from the oracle's own Alg. 2
(``oracle.sums_fwht`` per X-string), random numbers from ``sre_inputs.mc_streams`` (inputs).

  energy(psi, a)          f(X_a) = -ln(S(a) + eps), S(a) = sum_b <psi|X_a Z_b|psi>^4   (Eq. (17))
  ti_exact(psi, L)        <f>_beta by exact enumeration over all 2^N X-strings (Eq. (19)),
                          Simpson quadrature on beta_l = l/(L-1): the sampler's estimate with
                          zero Monte-Carlo error (SPEC's ti_sre_exact idea)
  mc_replay(...)          Alg. 3's chains, stepped one at a time in plain loops
"""
from __future__ import annotations

import math

import numpy as np

from . import sums_fwht


def energy(psi, a: int, epsilon: float = 0.0) -> float:
    s = float(sums_fwht(psi, [2.0], a_range=(int(a), int(a) + 1))[0])
    if s + epsilon <= 0.0:
        raise ValueError("S(a) + eps = 0")
    return -math.log(s + epsilon)


def all_energies(psi, epsilon: float = 0.0) -> np.ndarray:
    n = np.asarray(psi).size.bit_length() - 1
    _, pa = sums_fwht(psi, [2.0], per_a=True)
    s = pa[:, 0] + epsilon
    if np.any(s <= 0.0):
        raise ValueError("S(a) + eps = 0 for some a")
    assert s.size == 1 << n
    return -np.log(s)


def simpson(L: int):
    """Composite Simpson weights on beta_l = l/(L-1), l = 0..L-1 (L odd)."""
    if L < 3 or L % 2 == 0:
        raise ValueError("L must be odd and >= 3")
    h = 1.0 / (L - 1)
    w = []
    for l in range(L):
        if l == 0 or l == L - 1:
            w.append(h / 3.0)
        elif l % 2 == 1:
            w.append(4.0 * h / 3.0)
        else:
            w.append(2.0 * h / 3.0)
    return [l * h for l in range(L)], w


def mean_f_exact(f: np.ndarray, beta: float) -> float:
    """<f>_beta = sum_a Pi_beta(a) f(a), Pi_beta = e^{-beta f}/Z_beta (Eq. (18), (19)); the
    minimum is factored out of the exponent for range safety (it cancels in the ratio)."""
    g = np.exp(-beta * (f - f.min()))
    return float(np.sum(g * f) / np.sum(g))


def ti_exact(psi, L: int, epsilon: float = 0.0) -> float:
    """M_2 = -log2(e^{-I} - eps), I = sum_l w_l <f>_l: Eq. (M2_TI_reg_explicit_correct)
    written in reading C16's sign (I = ln Z_0 - ln Z_1, Z_0 = 2^N, Z_1 = S_2 + 2^N eps); = I / ln 2 at eps = 0."""
    f = all_energies(psi, epsilon)
    betas, w = simpson(L)
    integral = sum(wl * mean_f_exact(f, b) for b, wl in zip(betas, w))
    return -math.log2(math.exp(-integral) - epsilon)


def mc_replay(psi, L: int, streams, burn_in: int, n_samples: int, epsilon: float = 0.0):
    """Alg. 3 stepped literally: returns (mean_f[L], accepted[L], final patterns[L])."""
    init, flips, uni = streams
    betas, _ = simpson(L)
    cache = {}

    def f_of(a):
        if a not in cache:
            cache[a] = energy(psi, a, epsilon)
        return cache[a]

    means, accepted, final = [], [], []
    for l in range(L):
        a = int(init[l])
        fa = f_of(a)
        total, acc = 0.0, 0
        for step in range(burn_in + n_samples):
            prop = a
            for k in range(flips.shape[2]):
                prop ^= 1 << int(flips[step, l, k])
            fp = f_of(prop)
            p_acc = min(1.0, math.exp(-betas[l] * (fp - fa)))
            if uni[step, l] < p_acc:
                a, fa = prop, fp
                if step >= burn_in:
                    acc += 1
            if step >= burn_in:
                total += fa
        means.append(total / n_samples)
        accepted.append(acc)
        final.append(a)
    return np.array(means), np.array(accepted), np.array(final, dtype=np.uint64)
