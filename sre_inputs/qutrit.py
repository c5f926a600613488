"""Seeded synthetic qutrit states for the mana path (NEXT-3).  State preparation only: no
Wigner/mana arithmetic.  Index x = sum_j x_j 3^j (qutrit j is ternary digit j).

* ``haar(N, seed)``        -- i.i.d. complex Gaussian amplitudes, normalised (Haar on C^{3^N}).
* ``brickwall(N, depth)``  -- |0..0> evolved by layers of Haar U(9) gates on neighbouring
                              qutrits (the qutrit analogue of Eq. (46); the paper's mana workloads
                              are random-circuit states).
* ``zero``, ``strange``, ``kron`` -- closed-form cases; ``clifford_circuit`` applies random
  qutrit Clifford gates (F, S, SUM), under which mana is invariant.
"""
from __future__ import annotations

import math

import numpy as np

from . import haar_unitary

W = np.exp(2j * math.pi / 3)
F3 = np.array([[1, 1, 1], [1, W, W * W], [1, W * W, W]], dtype=np.complex128) / math.sqrt(3.0)
S3 = np.diag([1.0, 1.0, W]).astype(np.complex128)        # qutrit phase gate (Clifford)


def _normalise(psi):
    return psi / math.sqrt(float(np.sum(psi.real ** 2 + psi.imag ** 2)))


def haar(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    d = 3 ** n
    return _normalise((rng.standard_normal(d) + 1j * rng.standard_normal(d)).astype(np.complex128))


def zero(n: int) -> np.ndarray:
    psi = np.zeros(3 ** n, dtype=np.complex128)
    psi[0] = 1.0
    return psi


def strange() -> np.ndarray:
    return np.array([0.0, 1.0, -1.0], dtype=np.complex128) / math.sqrt(2.0)


def kron(states) -> np.ndarray:
    """Product state from single-qutrit states [q0, q1, ...] (q0 is the least significant digit)."""
    psi = np.ones(1, dtype=np.complex128)
    for q in states:
        psi = np.kron(np.asarray(q, dtype=np.complex128), psi)
    return psi


def apply_1q(psi, u, j):
    n = round(math.log(psi.size, 3))
    v = psi.reshape(3 ** (n - 1 - j), 3, 3 ** j)
    return np.einsum("ab,xby->xay", u, v).reshape(-1)


def apply_2q(psi, u, i, j):
    """9x9 unitary on qutrits (i, j), local basis index 3*x_i + x_j (i < j)."""
    n = round(math.log(psi.size, 3))
    v = psi.reshape([3] * n)              # axis k <-> qutrit n-1-k
    ai, aj = n - 1 - i, n - 1 - j
    v = np.moveaxis(v, (ai, aj), (0, 1))
    shp = v.shape
    v = (u @ v.reshape(9, -1)).reshape(shp)
    return np.moveaxis(v, (0, 1), (ai, aj)).reshape(-1)


def sum_gate(psi, c, t):
    """SUM (qutrit CNOT): |x_c, x_t> -> |x_c, x_t + x_c>."""
    n = round(math.log(psi.size, 3))
    idx = np.arange(psi.size)
    xc = (idx // 3 ** c) % 3
    xt = (idx // 3 ** t) % 3
    dst = idx + (((xt + xc) % 3) - xt) * 3 ** t
    out = np.empty_like(psi)
    out[dst] = psi
    del n
    return out


def brickwall(n: int, depth: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    psi = zero(n)
    for r in range(1, depth + 1):
        start = 0 if r % 2 == 1 else 1
        for i in range(start, n - 1, 2):
            psi = apply_2q(psi, haar_unitary(9, rng), i, i + 1)
    return psi


def clifford_circuit(psi, depth: int, rng):
    n = round(math.log(psi.size, 3))
    for _ in range(depth):
        for j in range(n):
            g = rng.integers(3)
            if g == 1:
                psi = apply_1q(psi, F3, j)
            elif g == 2:
                psi = apply_1q(psi, S3, j)
        perm = rng.permutation(n)
        for k in range(0, n - 1, 2):
            psi = sum_gate(psi, int(perm[k]), int(perm[k + 1]))
    return psi


def density(psi) -> np.ndarray:
    """|psi><psi| as a 3^N x 3^N array (rho[r, c] = psi_r conj(psi_c))."""
    return np.outer(psi, np.conj(psi))


def reduced(psi, n_keep: int) -> np.ndarray:
    """Tr_B |psi><psi| keeping qutrits 0..n_keep-1 (the low ternary digits; reading C21)."""
    n = round(math.log(psi.size, 3))
    phi = psi.reshape(3 ** (n - n_keep), 3 ** n_keep)        # phi[x_B, x_A]
    return phi.T @ np.conj(phi)                                # rho[r, c] = sum_b phi[b,r] conj(phi[b,c])


def mixed_strange(p: float) -> np.ndarray:
    s = strange()
    return p * np.outer(s, np.conj(s)) + (1.0 - p) * np.eye(3) / 3.0


def random_mixed(n: int, rank: int, seed: int) -> np.ndarray:
    """sum_k p_k |psi_k><psi_k| with Haar psi_k and Dirichlet weights p (rank <= 3^N)."""
    rng = np.random.default_rng(seed)
    p = rng.dirichlet(np.ones(rank))
    rho = np.zeros((3 ** n, 3 ** n), dtype=np.complex128)
    for k in range(rank):
        v = rng.standard_normal(3 ** n) + 1j * rng.standard_normal(3 ** n)
        v /= np.linalg.norm(v)
        rho += p[k] * np.outer(v, np.conj(v))
    return rho
