"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Tolerances (reading C7): raw sums S_alpha relative 1e-10, M_alpha absolute
1e-10, chi element-wise 1e-12 x max|chi|.
"""
import json
import math
import os

import numpy as np
import pytest

import sre_inputs as si

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def sre():
    import paper_2601_07824_b200 as m
    m.load()
    return m


def cuda(psi):
    return torch.from_numpy(np.ascontiguousarray(psi)).to("cuda")


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300)))


def gpu_sums(sre, psi, alphas, lo=None, hi=None):
    t = cuda(psi)
    n = t.shape[-1].bit_length() - 1
    lo = 0 if lo is None else lo
    hi = (1 << n) if hi is None else hi
    out = sre.partial_sums(t, lo, hi, alphas)
    torch.cuda.synchronize()
    return out.cpu().numpy()


ALPHAS = [0.5, 1.0, 1.5, 2.0, 3.0]


@pytest.mark.parametrize("n", list(range(1, 15)))
def test_full_sums_vs_oracle_all_paths(sre, oracle_lib, n):
    """single-pass kernels (N <= 14): every raw sum vs Alg. 2 oracle, 5 alphas (two sweeps)."""
    psi = si.haar(n, 1000 + n)
    al = ALPHAS if n <= 12 else [1.0, 2.0, 3.0]
    g = gpu_sums(sre, psi, al)[0]
    o = oracle_lib.sums_fwht(psi, al)
    assert rel(g[:-1], o[:-1]) < 1e-10
    assert abs(g[-1] - o[-1]) <= 1e-10 * max(1.0, abs(o[-1]))


@pytest.mark.parametrize("n", [15, 16, 17, 18, 19, 20, 21, 22, 23, 24, 25, 26])
def test_two_pass_ranges_vs_oracle(sre, oracle_lib, n):
    """two-pass path: sums over ragged X-string ranges (incl. a = 0 and unaligned ends) vs oracle."""
    psi = si.haar(n, 2000 + n)
    D = 1 << n
    ranges = [(0, 3), (D - 5, D), (D // 2 + 7, D // 2 + 12)] if n >= 21 else [(0, 37), (D - 29, D), (D // 3, D // 3 + 41)]
    al = [1.0, 2.0, 3.0] if n <= 20 else [2.0]
    for lo, hi in ranges:
        g = gpu_sums(sre, psi, al, lo, hi)[0]
        o = oracle_lib.sums_fwht(psi, al, a_range=(lo, hi))
        assert rel(g[:-1], o[:-1]) < 1e-10, (lo, hi)
        if 1.0 in al:
            assert abs(g[-1] - o[-1]) <= 1e-10 * abs(o[-1])


@pytest.mark.parametrize("n", [21, 22, 23, 24])
def test_streamed_production_batches_vs_oracle(sre, oracle_lib, n):
    """N = 21..24 at the production launch size: a full K-aligned batch (K = 64 at N = 21, 32 above)
    runs the radix-64 pass A (k_passAq) and pass B (k_passBr); a second range has an odd batch
    (kcount = 13) and a third covers an a_h with a high pivot.  Raw sums vs the Alg. 2 oracle at 1e-10 for alpha = 1, 2, 3."""
    psi = si.haar(n, 4100 + n)
    K = 64 if n == 21 else 32
    D = 1 << n
    ranges = [(5 * K * 4096 // K * K, 5 * K * 4096 // K * K + K), (D // 2 + 8 * 1024, D // 2 + 8 * 1024 + 13),
              (D - 2 * K, D - K)]
    for lo, hi in ranges:
        g = gpu_sums(sre, psi, [1.0, 2.0, 3.0], lo, hi)[0]
        o = oracle_lib.sums_fwht(psi, [1.0, 2.0, 3.0], a_range=(lo, hi))
        assert rel(g[:-1], o[:-1]) < 1e-10, (lo, hi)
        assert abs(g[-1] - o[-1]) <= 1e-10 * abs(o[-1]), (lo, hi)


@pytest.mark.parametrize("n", [1, 2, 5, 6, 10, 11, 13, 14, 15, 17, 20, 21, 23, 24])
def test_chi_elementwise(sre, oracle_lib, n):
    """chi_b(a) for every b, sampled a, element by element against the oracle's Alg. 2 transform.
    For N >= 15 the 8-aligned a >= 2^L run the production kernels of the sums (staged k_passA10s +
    k_passBt, streamed k_passAq + k_passBr), the others the generic head kernels."""
    psi = si.haar(n, 3000 + n)
    D = 1 << n
    rng = np.random.default_rng(n)
    a_list = sorted({0, 1, D - 1, *[int(x) for x in rng.integers(0, D, 3)]})
    if n >= 15:
        lo = 1 << (10 if n <= 20 else 12)
        a_list = sorted(set(a_list) | {lo, D - 8, *[8 * int(x) for x in rng.integers(lo // 8, D // 8, 3)]})
    if n >= 23:
        a_list = [a for a in a_list if a % 8 == 0 and a >= 4096][:3] + [1]
    t = cuda(psi)
    for a in a_list:
        g = sre.chi(t, a).cpu().numpy()
        o = oracle_lib.chi(psi, a)
        scale = max(np.max(np.abs(o)), 1e-300)
        assert np.max(np.abs(g - o)) < 1e-12 * scale, a


def test_config1_t_state_and_haar(sre, oracle_lib):
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    m, ln = sre.exact(cuda(si.t_state(8)), [1.0, 2.0, 3.0])
    for mi, k in zip(m, ["1", "2", "3"]):
        assert abs(mi - g["t_state_N8"][k]) < 1e-10
    assert abs(ln) < 1e-12
    psi = si.haar(8, 8001)
    m, ln = sre.exact(cuda(psi), [2.0])
    mo, lo = oracle_lib.sre(psi, [2.0], "brute")
    assert abs(m[0] - mo[0]) < 1e-10 and abs(ln - lo) < 1e-12


def test_paper_zero_state_bitwise(sre):
    """P:1145-1146 printed SRE=-0.0 lost_norm=0.0 for |0>^16."""
    gold = json.load(open(os.path.join(GOLD, "paper_zero_state.json")))
    m, ln = sre.exact(cuda(si.zero(gold["N"])), [gold["alpha"]])
    assert m[0] == 0.0 and math.copysign(1.0, m[0]) == -1.0
    assert ln == 0.0


def test_host_pointer_end_to_end(sre, oracle_lib):
    psi = si.haar(11, 77)
    m_host, _ = sre.exact(psi, [2.0, 3.0])          # numpy (host) -> copied inside the C call
    m_dev, _ = sre.exact(cuda(psi), [2.0, 3.0])
    assert m_host == m_dev
    mo, _ = oracle_lib.sre(psi, [2.0, 3.0], "fwht")
    assert max(abs(x - y) for x, y in zip(m_host, mo)) < 1e-10


def test_stabilizer_and_t_doped(sre, oracle_lib):
    for n in (6, 12, 16):
        psi = si.random_clifford_state(n, 2 * n, 40 + n)
        m, ln = sre.exact(cuda(psi), [1.0, 2.0, 3.0, 0.5])
        assert max(abs(x) for x in m) < 1e-10 and abs(ln) < 1e-12
    for t in (1, 3, 7):
        psi = si.t_doped(15, t, 20, 90 + t)
        m, _ = sre.exact(cuda(psi), [2.0, 3.0, 1.0])
        for mi, a in zip(m, [2.0, 3.0, 1.0]):
            assert abs(mi - oracle_lib.t_state_m(a, t)) < 1e-10


def test_sharded_ranges_sum_to_full(sre):
    """Sums over disjoint X-string shards add up to the single call (multi-GPU arithmetic)."""
    for n in (9, 13, 16):
        psi = si.haar(n, 555 + n)
        D = 1 << n
        full = gpu_sums(sre, psi, [2.0, 3.0])[0]
        for G in (2, 4, 8):
            parts = sum(gpu_sums(sre, psi, [2.0, 3.0], g * D // G, (g + 1) * D // G)[0] for g in range(G))
            assert rel(parts[:-1], full[:-1]) < 1e-13


def test_batched_config3_full(sre, oracle_lib):
    """BASELINE config 3 in full (256 x N=14 Clifford+T, the bench batch): every T-doped state against
    its closed form M_2 = t M_2(|T>), every interleaved state's sums over an X-string
    range against the oracle, and every lost_norm."""
    batch, ts = si.config3_batch(14, 256, 14000)
    m, ln = sre.exact_batched(cuda(batch), [2.0])
    assert np.max(np.abs(ln)) < 1e-10
    tdoped = [i for i in range(256) if ts[i] is not None]
    assert len(tdoped) == 128
    for i in tdoped:
        assert abs(m[i, 0] - oracle_lib.t_state_m(2.0, ts[i])) < 1e-10, i
    g = sre.partial_sums(cuda(batch), 100, 132, [2.0]).cpu().numpy()
    for i in range(256):
        if ts[i] is None:
            o = oracle_lib.sums_fwht(batch[i], [2.0], a_range=(100, 132))
            assert rel(g[i, :2], o[:2]) < 1e-10, i


def test_scrambled_pair_n20(sre, oracle_lib):
    """Exact pin for a generic entangled N=20 state: M(C(psi10 (x) phi10)) = M(psi10) + M(phi10)."""
    lo, hi = si.haar(10, 2401), si.haar(10, 2402)
    psi = si.scrambled_pair(lo, hi, 6, 2403)
    m, ln = sre.exact(cuda(psi), [2.0])
    ref = oracle_lib.sre(lo, [2.0])[0][0] + oracle_lib.sre(hi, [2.0])[0][0]
    assert abs(m[0] - ref) < 1e-10
    assert abs(ln) < 1e-10


def test_error_paths(sre):
    psi = cuda(si.haar(6, 1))
    with pytest.raises(sre.SreError) as e:
        sre.exact(psi * 1.01, [2.0])
    assert e.value.code == 3
    with pytest.raises(sre.SreError) as e:
        sre.exact(psi, [0.0])
    assert e.value.code == 1
    with pytest.raises(sre.SreError) as e:
        sre.exact(psi, [float("nan")])
    assert e.value.code == 1
    with pytest.raises(sre.SreError) as e:
        sre.partial_sums(psi, 5, 3, [2.0])
    assert e.value.code == 2
    with pytest.raises(sre.SreError) as e:
        sre.partial_sums(psi, 0, 65, [2.0])
    assert e.value.code == 2


def test_config2_full_vs_frozen_oracle(sre):
    """BASELINE config 2 (N=16 Haar, alpha in {1,2,3}) in full against the oracle's frozen sums
    (tests/golden/oracle_c2.json, written by tools/make_fixtures.py from oracle/ only)."""
    import hashlib
    g = json.load(open(os.path.join(GOLD, "oracle_c2.json")))
    psi = si.haar(g["n"], g["seed"])
    assert hashlib.sha256(psi.tobytes()).hexdigest() == g["psi_sha256"]
    s = gpu_sums(sre, psi, g["alphas"])[0]
    assert rel(s[:-1], g["sums"][:-1]) < 1e-10
    assert abs(s[-1] - g["sums"][-1]) <= 1e-10 * abs(g["sums"][-1])
    m, ln = sre.exact(cuda(psi), g["alphas"])
    assert max(abs(a - b) for a, b in zip(m, g["M"])) < 1e-10
    assert abs(ln) < 1e-10


def test_config5_n24_sampled_and_t_state(sre, oracle_lib):
    """BASELINE config 5 size (N=24): sampled X-string ranges vs the oracle, and |T>^24 per
    X-string closed form (product state: S_a = prod_j s_j(a_j) with s(0) = 1 + 0, s(1) = 2 (1/2)^alpha)."""
    n = 24
    psi = si.haar(n, 24001)
    for lo, hi in ((123456, 123460), ((1 << 24) - 3, 1 << 24)):
        g = gpu_sums(sre, psi, [2.0], lo, hi)[0]
        o = oracle_lib.sums_fwht(psi, [2.0], a_range=(lo, hi))
        assert rel(g[:2], o[:2]) < 1e-10
    t = si.t_state(n)
    for a in (0, 1, 0xABCDE, (1 << 24) - 1):
        g = gpu_sums(sre, t, [2.0], a, a + 1)[0]
        w = bin(a).count("1")
        expect = (1.0 ** 2) ** (n - w) * (2 * 0.5 ** 2.0) ** w   # <I>,<Z>: (1, 0); <X>,<Y>: 1/sqrt2 each
        assert abs(g[0] - expect) <= 1e-12 * expect


@pytest.mark.parametrize("n", [3, 8, 12, 14, 16, 20, 22])
def test_fp32_mode_vs_oracle(sre, oracle_lib, n):
    """Optional FP32 mode (north star): FP32 transform, FP64 accumulation, S_alpha within 1e-4."""
    psi = si.haar(n, 4000 + n)
    D = 1 << n
    lo, hi = (0, D) if n <= 12 else ((D // 2 + 13, D // 2 + 13 + 40) if n < 22 else (D // 2 + 8, D // 2 + 12))
    al = [1.0, 2.0, 3.0] if n <= 16 else [2.0]
    t = cuda(psi)
    g = sre.partial_sums(t, lo, hi, al, precision="fp32").cpu().numpy()[0]
    o = oracle_lib.sums_fwht(psi, al, a_range=(lo, hi))
    assert rel(g[:-1], o[:-1]) < 1e-4
    if 1.0 in al:
        assert abs(g[-1] - o[-1]) <= 1e-4 * abs(o[-1])
    if n <= 14:
        m32, _ = sre.exact(t, [2.0], precision="fp32")
        m64, _ = sre.exact(t, [2.0])
        assert abs(m32[0] - m64[0]) < 1e-4 * max(1.0, abs(m64[0]))


def test_exact_resumable_matches_exact(sre, tmp_path):
    from paper_2601_07824_b200.resume import exact_resumable
    psi = cuda(si.haar(16, 99))
    j = str(tmp_path / "j.json")
    assert exact_resumable(psi, [2.0], chunk=4096, journal_path=j, max_chunks=5) is None
    m, ln = exact_resumable(psi, [2.0], chunk=4096, journal_path=j)
    m0, ln0 = sre.exact(psi, [2.0])
    assert abs(m[0] - m0[0]) < 1e-12 and abs(ln - ln0) < 1e-12


def _sums_in_subprocess(env_extra, n, seed, lo, hi, alphas, batch=0):
    """partial_sums in a fresh process (the kernel-variant switches are read once per process)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    gen = f"si.haar_batch({n}, {batch}, {seed})" if batch else f"si.haar({n}, {seed})"
    code = ("import numpy as np, torch, sre_inputs as si, paper_2601_07824_b200 as sre; "
            f"psi = torch.from_numpy({gen}).cuda(); "
            f"print(repr(sre.partial_sums(psi, {lo}, {hi}, {alphas!r}).cpu().numpy().tolist()))")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, **env_extra),
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    return np.array(eval(out.stdout.strip().splitlines()[-1]))


@pytest.mark.parametrize("env,n,lo,hi,batch", [
    ({"SRE_MIDR": "0"}, 14, 0, 1 << 14, 4),          # k_midr ring-fed generation vs k_mid's L2 gathers
    ({"SRE_PAW_TMA": "0"}, 22, 4096, 4096 + 256, 0),   # k_passAw TMA-store exit vs coalesced STG exit
])
def test_kernel_variants_bitwise(sre, env, n, lo, hi, batch):
    """The round-2 variants move the same values by other means (bulk-copy ring instead of gathers,
    TMA tensor store instead of STG); grids and accumulation order are unchanged, so the raw sums
    are bitwise those of the variant they replace."""
    alphas = [1.0, 2.0, 3.0]
    a = _sums_in_subprocess({}, n, 4242, lo, hi, alphas, batch)
    b = _sums_in_subprocess(env, n, 4242, lo, hi, alphas, batch)
    assert np.array_equal(a, b)
