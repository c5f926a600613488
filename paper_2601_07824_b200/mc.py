"""Thermodynamic-integration Monte-Carlo estimate of M_2 (Sec. 3.2.2-3.2.4, Alg. 3).

The L chains (one per grid point beta_l) advance in lockstep; each step proposes one move per
chain and evaluates all L proposal energies with ONE batched call into the CUDA library
(``sre_x_string_sums``: per X-string S(a) = sum_b <psi|X_a Z_b|psi>^4 from the same fused
generation + Walsh-Hadamard + power-sum kernels as the exact path).  The host does only the
Metropolis bookkeeping.

Readings (C15-C17):
  C15 f(X_a) = -ln(S(a) + eps): natural log (Eq. (17) prints log2, but Z_1 = sum_a e^{-f} = S_2 + 2^N eps
      in the text below it requires ln).
  C16 sign: <f>_beta = -d ln Z / d beta gives  int_0^1 <f> dbeta = ln Z_0 - ln Z_1 (Eq. (20) prints the
      opposite), so M_2 = +(1/ln 2) sum_l w_l <f>_l  (Alg. 3's return line carries the other sign);
      checked against |T>^N, where the integral is N log2(4/3) in closed form.
  C17 grid: beta_l = l/(L-1), l = 0..L-1 with composite Simpson weights, which need odd L (Alg. 3
      asks for an even number of points with Simpson weights).
"""
from __future__ import annotations

import math

import numpy as np


def simpson_weights(L: int) -> np.ndarray:
    if L < 3 or L % 2 == 0:
        raise ValueError("composite Simpson needs an odd number of grid points L >= 3 (reading C17)")
    w = np.ones(L)
    w[1:-1:2] = 4.0
    w[2:-1:2] = 2.0
    return w / (3.0 * (L - 1))


def energies(psi, a_list, epsilon: float = 0.0, workspace=None):
    """f(X_a) = -ln(S(a) + eps) for every a in a_list (one batched library call)."""
    from . import x_string_sums
    s = x_string_sums(psi, np.asarray(a_list, dtype=np.uint64), [2.0], workspace=workspace)[:, 0].cpu().numpy()
    s = s + epsilon
    if np.any(s <= 0.0):
        raise ValueError("S(a) + eps = 0 for a proposed X-string: use epsilon > 0 (P:565-580)")
    return -np.log(s)


def mc_sre(psi, L: int = 21, n_samples: int = 1000, burn_in: int | None = None, streams=None,
           epsilon: float = 0.0):
    """Alg. 3: returns dict(m2, stderr, mean_f[L], var_f[L], acc_rate[L], betas, weights).
    stderr follows Eq. (27)/(28) with per-chain variances of the mean from batch means.
    streams = (init[L], flips[steps, L, width], uniforms[steps, L]): the random numbers of the chains,
    drawn by the caller (the product draws none itself)."""
    import torch

    n = psi.shape[-1].bit_length() - 1
    burn = 10 * n if burn_in is None else burn_in
    steps = burn + n_samples
    if streams is None:
        raise ValueError("streams=(init, flips, uniforms) is required: the sampler consumes random numbers drawn "
                         "by the caller (e.g. sre_inputs.mc_streams(seed, L, burn_in + n_samples, N, move_width))")
    init, flips, uni = streams
    betas = np.linspace(0.0, 1.0, L)
    w = simpson_weights(L)
    ws = None
    from . import workspace_size
    ws = torch.empty(workspace_size(n, 1, 1), dtype=torch.uint8, device=psi.device)
    a = init.astype(np.uint64).copy()
    f = energies(psi, a, epsilon, ws)
    hist = np.zeros((n_samples, L))
    acc = np.zeros(L)
    one = np.uint64(1)
    for step in range(steps):
        prop = a.copy()
        for k in range(flips.shape[2]):
            prop ^= np.left_shift(one, flips[step, :, k].astype(np.uint64))
        fp = energies(psi, prop, epsilon, ws)
        accept = uni[step] < np.exp(np.minimum(0.0, -betas * (fp - f)))
        a = np.where(accept, prop, a)
        f = np.where(accept, fp, f)
        if step >= burn:
            hist[step - burn] = f
            acc += accept
    mean_f = hist.mean(axis=0)
    nb = max(2, int(math.isqrt(n_samples)))
    bsz = n_samples // nb
    bm = hist[: nb * bsz].reshape(nb, bsz, L).mean(axis=1)
    var_mean = bm.var(axis=0, ddof=1) / nb
    # Eq. (M2_TI_reg_explicit_correct), in reading C16's sign: I = sum_l w_l <f>_l = ln Z_0 - ln Z_1
    # with Z_1 = S_2 + 2^N eps, so M_2 = -log2(e^{-I} - eps) (= I / ln 2 at eps = 0); the error propagates
    # with dM_2/dI = e^{-I} / ((e^{-I} - eps) ln 2) (Eq. (m2error), at eps = 0)
    integral = float(np.dot(w, mean_f))
    z = math.exp(-integral) - epsilon
    if z <= 0.0:
        raise ValueError("e^{-I} <= eps: the estimate is outside the regularised range (P:469-474)")
    m2 = -math.log2(z)
    stderr = float(math.sqrt(np.dot(w * w, var_mean)) * math.exp(-integral) / (z * math.log(2.0)))
    return {"m2": m2, "stderr": stderr, "mean_f": mean_f, "var_f": hist.var(axis=0), "acc_rate": acc / n_samples,
            "betas": betas, "weights": w, "final_patterns": a}
