"""GPU parity for mixed-state qutrit mana (NEXT-4): csrc/mana_mixed.cu through the C ABI against
the Alg. 6 oracle (oracle/mana.py, long double) on the same seeded density matrices, every leg
plan the planner can produce, and closed forms at the maximum size N_A = 10 (56 GB on device).
Tolerance rtol 1e-11 on both sums (FP64 leg transforms)."""
import math
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
RTOL = 1e-11


@pytest.fixture(scope="module")
def qm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_07824_b200 import qutrit
    return qutrit


def _sums(qm, rho):
    import torch
    flat = torch.from_numpy(np.ascontiguousarray(rho.flatten(order="F"))).cuda()
    n = round(math.log(rho.shape[0], 3))
    return qm.mixed_sums_(flat, n).cpu().numpy()


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 7, 8])
def test_vs_alg6_oracle(qm, n):
    from oracle import mana as om
    import sre_inputs.qutrit as q
    rho = q.random_mixed(n, 3, 900 + n)
    ref = om.sums_mixed_alg6(rho)
    np.testing.assert_allclose(_sums(qm, rho), ref, rtol=RTOL)
    m, tr = qm.mana_mixed(rho)
    assert m == pytest.approx(math.log2(ref[0] / 3 ** n), abs=1e-12) and tr == pytest.approx(1.0, abs=1e-12)


@pytest.mark.parametrize("plan", ["0:3,3:2,3:2", "0:2,2:3,2:2", "0:3,3:2,3:1,3:1", "0:4,2:1,3:2", "0:4,4:2,4:1", "0:1,0:3,2:3"])
def test_leg_plans(qm, plan, monkeypatch):
    """Every (SP, NL) kernel instance: the planner override SRE_MIXED_PLAN must give the same sums."""
    from oracle import mana as om
    import sre_inputs.qutrit as q
    rho = q.random_mixed(7, 2, 950)
    ref = om.sums_mixed_alg6(rho)
    monkeypatch.setenv("SRE_MIXED_PLAN", plan)
    np.testing.assert_allclose(_sums(qm, rho), ref, rtol=RTOL)


@pytest.mark.parametrize("n", [5, 6, 8])
def test_tma_tile_passes_vs_ldg(qm, n, monkeypatch):
    """k_legs_tma (TMA tiles) and the LDG/STG k_legs apply the same leg9 to the same fibers in the
    same leg order; only the final pass's per-CTA accumulation order differs (other grid), so the
    sums agree to a few ulps of the sum, and both with the oracle."""
    from oracle import mana as om
    import sre_inputs.qutrit as q
    rho = q.random_mixed(n, 2, 970 + n)
    monkeypatch.setenv("SRE_MIXED_TMA", "1")
    a = _sums(qm, rho)
    monkeypatch.setenv("SRE_MIXED_TMA", "0")
    b = _sums(qm, rho)
    np.testing.assert_allclose(a, b, rtol=1e-14)
    np.testing.assert_allclose(a, om.sums_mixed_alg6(rho), rtol=RTOL)


def test_pure_state_matches_alg5_path(qm):
    """rho = |psi><psi| at N = 9 (6.2 GB): the mixed path equals the pure-state path (both GPU,
    the pure one parity-tested against its own oracle)."""
    import sre_inputs.qutrit as q
    psi = q.brickwall(9, 4, 960)
    m_pure, _ = qm.mana(psi)
    m_mix, tr = qm.mana_mixed(q.density(psi))
    assert m_mix == pytest.approx(m_pure, abs=1e-11) and tr == pytest.approx(1.0, abs=1e-12)


def test_reduced_state_paper_workflow(qm):
    """N = 10 brick-wall state (depth 3), reduced to N_A = 8 (657 MiB); oracle Alg. 6
    at N_A = 8 and the monotonicity bound mana(rho_A) <= mana(psi)."""
    from oracle import mana as om
    import sre_inputs.qutrit as q
    psi = q.brickwall(10, 3, 970)
    rho = q.reduced(psi, 8)
    ref = om.sums_mixed_alg6(rho)
    np.testing.assert_allclose(_sums(qm, rho), ref, rtol=RTOL)
    m, _ = qm.mana_mixed(rho)
    assert 0.0 < m <= qm.mana(psi)[0] + 1e-12


def test_max_size_closed_forms(qm):
    """N_A = 10 (9^10 x 16 B = 56 GB, built on the device): a product of strange-state mixtures
    with p_k in [0, 1] has mana sum_k log2(max(1, (7 + 8 p_k)/9)); I/3^10 has mana 0."""
    import torch
    import sre_inputs.qutrit as q
    from oracle import mana as om
    ps = [1.0, 0.9, 0.2, 0.6, 1.0, 0.35, 0.0, 0.75, 1.0, 0.5]
    rho = torch.ones((1, 1), dtype=torch.complex128, device="cuda")
    for p in ps:                                   # qutrit k = digit k: kron(new, old)
        rho = torch.kron(torch.from_numpy(q.mixed_strange(p)).cuda(), rho)
    flat = rho.t().contiguous().view(-1)
    del rho
    s = qm.mixed_sums_(flat, 10).cpu().numpy()
    expect = sum(om.mixed_strange_mana(p) for p in ps)
    assert math.log2(s[0] / 3 ** 10) == pytest.approx(expect, abs=1e-10)
    assert s[1] / 3 ** 10 == pytest.approx(1.0, abs=1e-10)
    flat.zero_()
    d = 3 ** 10
    flat[:: d + 1] = 1.0 / d                       # I / 3^N (column-major diagonal)
    s = qm.mixed_sums_(flat, 10).cpu().numpy()
    assert s[0] / d == pytest.approx(1.0, abs=1e-10)
    del flat
    torch.cuda.empty_cache()


def test_determinism_and_errors(qm):
    import ctypes

    import torch
    from paper_2601_07824_b200 import SreError
    import sre_inputs.qutrit as q
    rho = q.random_mixed(6, 4, 990)
    a, b = _sums(qm, rho), _sums(qm, rho)
    np.testing.assert_allclose(a, b, rtol=1e-14)
    with pytest.raises(SreError) as e:
        qm.mana_mixed(2.0 * rho)
    assert e.value.code == 3
    lib = qm._lib()
    host = np.zeros(81, dtype=np.complex128)
    ws = torch.empty(qm._lib().sre_mana_mixed_workspace_size(2), dtype=torch.uint8, device="cuda")
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    assert lib.sre_mana_mixed_sums(ctypes.c_void_p(host.ctypes.data), 2, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                   ctypes.c_void_p(out.data_ptr()), None) == 1
    dev = torch.zeros(81, dtype=torch.complex128, device="cuda")
    assert lib.sre_mana_mixed_sums(ctypes.c_void_p(dev.data_ptr()), 11, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                   ctypes.c_void_p(out.data_ptr()), None) == 2
    assert lib.sre_mana_mixed_sums(ctypes.c_void_p(dev.data_ptr()), 2, ctypes.c_void_p(ws.data_ptr()), 100,
                                   ctypes.c_void_p(out.data_ptr()), None) == 4
