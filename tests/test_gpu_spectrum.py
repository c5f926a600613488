"""GPU parity for the spectrum epilogue (NEXT-2): histogram of |<P>|^2 from the single-pass
kernels against the oracle (oracle.spectrum, Alg. 2 chi per X-string) and the |T>^N closed
form.  Integer counts: compared exactly (DESIGN C22)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sre():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2601_07824_b200 as m
    return m


def _cuda(psi):
    import torch
    return torch.from_numpy(np.ascontiguousarray(psi)).cuda()


@pytest.mark.parametrize("n", [1, 2, 4, 6, 9, 12, 14])
def test_t_state_closed_form(sre, n):
    import oracle
    import sre_inputs as si
    np.testing.assert_array_equal(sre.spectrum(_cuda(si.t_state(n))), oracle.t_state_spectrum(n))


@pytest.mark.parametrize("n", [3, 7, 11])
def test_vs_oracle(sre, n):
    import oracle
    import sre_inputs as si
    psi = si.brickwall(n, 3, 1300 + n) if n > 3 else si.haar(n, 1300)
    got = sre.spectrum(_cuda(psi))
    ref = oracle.spectrum(psi) if n <= 7 else oracle.spectrum(psi, (0, 64))
    if n > 7:
        got = sre.spectrum(_cuda(psi), 0, 64)
    np.testing.assert_array_equal(got, ref)


def test_ranges_and_errors(sre):
    import sre_inputs as si
    from paper_2601_07824_b200 import SreError
    psi = _cuda(si.haar(12, 1400))
    whole = sre.spectrum(psi)
    assert whole.sum() == 4 ** 12
    k = 1234
    np.testing.assert_array_equal(sre.spectrum(psi, 0, k) + sre.spectrum(psi, k, 1 << 12), whole)
    assert sre.spectrum(psi, 5, 5).sum() == 0
    with pytest.raises(SreError) as e:
        sre.spectrum(psi, 10, 5000)
    assert e.value.code == 2


@pytest.mark.parametrize("n", [15, 16, 21])
def test_t_state_two_pass(sre, n):
    """Pass-B epilogues (staged N = 15-20, streamed N = 21-25, generic heads a < 1024)."""
    import oracle
    import sre_inputs as si
    np.testing.assert_array_equal(sre.spectrum(_cuda(si.t_state(n))), oracle.t_state_spectrum(n))


@pytest.mark.parametrize("lo,hi", [(0, 24), (2048, 2080), (1021, 1043)])
def test_two_pass_vs_oracle(sre, lo, hi):
    """N = 16 brick-wall: generic heads, aligned staged groups and a range straddling both."""
    import oracle
    import sre_inputs as si
    psi = si.brickwall(16, 3, 1500)
    np.testing.assert_array_equal(sre.spectrum(_cuda(psi), lo, hi), oracle.spectrum(psi, (lo, hi)))
