"""NEXT-1 on the GPU: per-X-string energies through the C ABI vs the oracle, and the sampler's
chains vs the oracle's replay on the same random streams."""
import math

import numpy as np
import pytest

import sre_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sre():
    import paper_2601_07824_b200 as m
    m.load()
    return m


@pytest.mark.parametrize("n", [2, 5, 12, 16, 20])
def test_x_string_sums_vs_oracle(sre, oracle_lib, n):
    psi = si.haar(n, 6000 + n)
    rng = np.random.default_rng(n)
    a = rng.integers(0, 1 << n, size=12).astype(np.uint64)
    a[3] = a[7]                                   # repeats allowed
    a[0] = 0
    g = sre.x_string_sums(torch.from_numpy(psi).cuda(), a, [1.0, 2.0, 3.0]).cpu().numpy()
    for i, ai in enumerate(a):
        o = oracle_lib.sums_fwht(psi, [1.0, 2.0, 3.0], a_range=(int(ai), int(ai) + 1))
        assert np.max(np.abs(g[i, :-1] - o[:-1]) / np.maximum(np.abs(o[:-1]), 1e-300)) < 1e-10
        assert abs(g[i, -1] - o[-1]) <= 1e-10 * max(1.0, abs(o[-1]))


def test_sampler_matches_oracle_replay(sre):
    import oracle.mc as omc
    from paper_2601_07824_b200 import mc
    n, L, burn, ns = 8, 5, 20, 300
    psi = si.haar(n, 71)
    streams = si.mc_streams(9, L, burn + ns, n)
    r = mc.mc_sre(torch.from_numpy(psi).cuda(), L=L, n_samples=ns, burn_in=burn, streams=streams)
    means, acc, final = omc.mc_replay(psi, L, streams, burn, ns)
    assert np.max(np.abs(r["mean_f"] - means)) < 1e-9
    assert np.array_equal(np.round(r["acc_rate"] * ns).astype(int), acc)
    assert np.array_equal(r["final_patterns"], final)


def test_sampler_estimates_exact_m2(sre, oracle_lib):
    """The paper's MC workload: shallow brick-wall circuits, where S(a) varies
    smoothly with the support of a.  (For fully Haar states Pi_1 puts ~1/4 of its mass on the
    single pattern a = 0, which single-flip chains rarely reach -- DESIGN.md NEXT-1.)"""
    import oracle.mc as omc
    from paper_2601_07824_b200 import mc
    n, L = 12, 11
    psi = si.brickwall(n, 2, 72)
    t = torch.from_numpy(psi).cuda()
    exact = sre.exact(t, [2.0])[0][0]
    quad = omc.ti_exact(psi, L)                   # same quadrature, zero MC error
    r = mc.mc_sre(t, L=L, n_samples=2000, streams=si.mc_streams(5, L, 10 * n + 2000, n, 1))
    assert abs(quad - exact) < 0.05
    assert abs(r["m2"] - quad) < 6 * r["stderr"] + 1e-3
    assert r["acc_rate"][0] == 1.0
