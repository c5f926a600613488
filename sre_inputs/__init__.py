"""Seeded synthetic input states shared by the oracle-side tests and the CUDA path.

This module prepares state vectors only; it holds none of the SRE arithmetic (no Pauli
expectations, no Hadamard transform, no power sums).  Both sides receive the same numpy
array.  Recipes:

* ``haar(N, seed)``       -- i.i.d. complex Gaussian amplitudes, normalised: exactly Haar on the
                             unit sphere (reading C9; the paper's workloads are deep random
                             circuits whose states approach this).
* ``brickwall(N, depth)`` -- the paper's generator, Eq. (46): |0..0> evolved by
                             layers of Haar-random two-qubit gates on a 1-D open chain.
* ``zero(N)``, ``t_state(N)``, ``product(N, seed)`` -- closed-form cases.
* ``clifford_circuit`` / ``t_doped`` / ``clifford_t`` / ``scrambled_pair`` -- Clifford(+T)
  circuits from {H, S, CNOT, T} applied to a state vector (BASELINE config 3, reading C10).

Conventions: amplitude index x = sum_j x_j 2^j, i.e. qubit j is bit j (LSB = qubit 0).
Random numbers come from numpy's PCG64 (``np.random.default_rng(seed)``).
"""
from __future__ import annotations

import math

import numpy as np

_H = np.array([[1.0, 1.0], [1.0, -1.0]], dtype=np.complex128) / math.sqrt(2.0)
_S = np.array([[1.0, 0.0], [0.0, 1.0j]], dtype=np.complex128)
_T = np.array([[1.0, 0.0], [0.0, np.exp(1j * math.pi / 4)]], dtype=np.complex128)


def _normalise(psi: np.ndarray) -> np.ndarray:
    return psi / math.sqrt(float(np.sum(psi.real ** 2 + psi.imag ** 2)))


def haar(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    d = 1 << n
    psi = rng.standard_normal(d) + 1j * rng.standard_normal(d)
    return _normalise(psi.astype(np.complex128))


def haar_batch(n: int, b: int, seed: int) -> np.ndarray:
    return np.stack([haar(n, seed * 100003 + i) for i in range(b)])


def zero(n: int) -> np.ndarray:
    psi = np.zeros(1 << n, dtype=np.complex128)
    psi[0] = 1.0
    return psi


def kron_qubits(states) -> np.ndarray:
    """Product state from single-qubit states [q0, q1, ...] (q0 is the least significant bit)."""
    psi = np.ones(1, dtype=np.complex128)
    for q in states:
        psi = np.kron(np.asarray(q, dtype=np.complex128), psi)
    return psi


def t_state(n: int) -> np.ndarray:
    t = np.array([1.0, np.exp(1j * math.pi / 4)], dtype=np.complex128) / math.sqrt(2.0)
    return kron_qubits([t] * n)


def product(n: int, seed: int):
    """Random product state; returns (psi, bloch) with bloch[j] = (<X>, <Y>, <Z>) of qubit j."""
    rng = np.random.default_rng(seed)
    qs, bloch = [], []
    for _ in range(n):
        q = rng.standard_normal(2) + 1j * rng.standard_normal(2)
        q = q / np.linalg.norm(q)
        a, b = q
        bloch.append((2 * (np.conj(a) * b).real, 2 * (np.conj(a) * b).imag, abs(a) ** 2 - abs(b) ** 2))
        qs.append(q)
    return kron_qubits(qs), bloch


def apply_1q(psi: np.ndarray, u: np.ndarray, j: int) -> np.ndarray:
    n = psi.size.bit_length() - 1
    v = psi.reshape(1 << (n - 1 - j), 2, 1 << j)
    return np.einsum("ab,xby->xay", u, v).reshape(-1)


def apply_cnot(psi: np.ndarray, c: int, t: int) -> np.ndarray:
    idx = np.arange(psi.size)
    src = np.where((idx >> c) & 1, idx ^ (1 << t), idx)
    return psi[src]


def apply_2q(psi: np.ndarray, u: np.ndarray, i: int, j: int) -> np.ndarray:
    """Apply a 4x4 unitary on qubits (i, j); basis order |q_i q_j> with q_i the high bit."""
    n = psi.size.bit_length() - 1
    idx = np.arange(psi.size)
    out = np.zeros_like(psi)
    sub = ((idx >> i) & 1) * 2 + ((idx >> j) & 1)
    base = idx & ~((1 << i) | (1 << j))
    for r in range(4):
        mask = sub == r
        acc = np.zeros(int(mask.sum()), dtype=np.complex128)
        b = base[mask]
        for c in range(4):
            src = b | (((c >> 1) & 1) << i) | ((c & 1) << j)
            acc += u[r, c] * psi[src]
        out[mask] = acc
    del n
    return out


def haar_unitary(d: int, rng) -> np.ndarray:
    """Haar-random U(d) via QR of a complex Ginibre matrix with the phase fix (Mezzadri)."""
    z = (rng.standard_normal((d, d)) + 1j * rng.standard_normal((d, d))) / math.sqrt(2.0)
    q, r = np.linalg.qr(z)
    ph = np.diag(r) / np.abs(np.diag(r))
    return q * ph


def brickwall(n: int, depth: int, seed: int) -> np.ndarray:
    """Eq. (46): U_t = prod_r U^(r), odd layers on bonds (0,1),(2,3),..., even layers on
    (1,2),(3,4),... (open chain, reading of S:227), each gate Haar on U(4)."""
    rng = np.random.default_rng(seed)
    psi = zero(n)
    for r in range(1, depth + 1):
        start = 0 if r % 2 == 1 else 1
        for i in range(start, n - 1, 2):
            psi = apply_2q(psi, haar_unitary(4, rng), i, i + 1)
    return psi


def clifford_circuit(psi: np.ndarray, depth: int, rng) -> np.ndarray:
    """depth layers of {I,H,S} on every qubit followed by CNOTs on a random perfect matching."""
    n = psi.size.bit_length() - 1
    for _ in range(depth):
        for j in range(n):
            g = rng.integers(3)
            if g == 1:
                psi = apply_1q(psi, _H, j)
            elif g == 2:
                psi = apply_1q(psi, _S, j)
        perm = rng.permutation(n)
        for k in range(0, n - 1, 2):
            c, t = int(perm[k]), int(perm[k + 1])
            if rng.integers(2):
                c, t = t, c
            psi = apply_cnot(psi, c, t)
    return psi


def random_clifford_state(n: int, depth: int, seed: int) -> np.ndarray:
    return clifford_circuit(zero(n), depth, np.random.default_rng(seed))


def t_doped(n: int, t: int, depth: int, seed: int) -> np.ndarray:
    """|T>^{(x)t} (x) |0>^{(x)(N-t)} followed by a random Clifford circuit: M_alpha = t M_alpha(|T>)."""
    tq = np.array([1.0, np.exp(1j * math.pi / 4)], dtype=np.complex128) / math.sqrt(2.0)
    z = np.array([1.0, 0.0], dtype=np.complex128)
    psi = kron_qubits([tq] * t + [z] * (n - t))
    return clifford_circuit(psi, depth, np.random.default_rng(seed))


def clifford_t(n: int, layers: int, seed: int) -> np.ndarray:
    """Interleaved Clifford+T: after every Clifford layer, a T gate on a random qubit."""
    rng = np.random.default_rng(seed)
    psi = zero(n)
    for _ in range(layers):
        psi = clifford_circuit(psi, 1, rng)
        psi = apply_1q(psi, _T, int(rng.integers(n)))
    return psi


def scrambled_pair(psi_lo: np.ndarray, psi_hi: np.ndarray, depth: int, seed: int) -> np.ndarray:
    """C (psi_hi (x) psi_lo) with C a random Clifford circuit: M = M(psi_lo) + M(psi_hi) exactly
    (additivity + Clifford invariance)."""
    return clifford_circuit(np.kron(psi_hi, psi_lo), depth, np.random.default_rng(seed))


def config3_batch(n: int = 14, b: int = 256, seed: int = 14000):
    """BASELINE config 3: b states of N qubits from seeded Clifford+T circuits (reading C10):
    the first b/2 are T-doped Clifford states with t = i mod 15 (exact M = t M(|T>)); the rest
    are interleaved Clifford+T circuits with 2N layers.  Returns (batch [b, 2^N], t_counts list
    with None for the interleaved ones)."""
    states, ts = [], []
    for i in range(b):
        if i < b // 2:
            t = i % 15
            states.append(t_doped(n, min(t, n), 2 * n, seed + i))
            ts.append(min(t, n))
        else:
            states.append(clifford_t(n, 2 * n, seed + i))
            ts.append(None)
    return np.stack(states), ts


def mc_streams(seed: int, n_chains: int, n_steps: int, n_qubits: int, move_width: int = 1):
    """Random numbers drawn by the thermodynamic-integration sampler (Alg. 3), generated
    up front so the CUDA-path sampler and the oracle's replay consume the identical stream:
      init    [n_chains]                  initial X-pattern of each beta-chain (uniform in [0, 2^N))
      flips   [n_steps, n_chains, width]  qubit positions whose a-bit the proposal flips
      uniform [n_steps, n_chains]         U(0,1) for the Metropolis acceptance test
    (holds no SRE arithmetic)."""
    rng = np.random.default_rng(seed)
    init = rng.integers(0, 1 << n_qubits, size=n_chains, dtype=np.uint64)
    flips = rng.integers(0, n_qubits, size=(n_steps, n_chains, move_width))
    uniform = rng.random((n_steps, n_chains))
    return init, flips, uniform
