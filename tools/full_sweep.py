"""Full exact sweep at large N on one GPU, with its exact pin and a clock record.

    python tools/full_sweep.py N {scrambled|haar} [chunk_log2] > log

scrambled: psi = C (phi_hi (x) phi_lo), phi = Haar states of N/2 qubits (seeds 24002/24003 at N = 24),
           C a depth-6 random Clifford circuit (seed 24004).  Additivity and Clifford invariance
            fix M_2(psi) = M_2(phi_lo) + M_2(phi_hi) exactly; the halves come from
           the CPU oracle (oracle/, Alg. 2 in long double).  This is the production-size parity pin of
           SURVEY.md section 8(c) C5.
haar:      BASELINE config 5's state (seed 24001 at N = 24); sanity |M_2 - (log2(2^N + 3) - 2)| < 40 2^-N.
Every X-string runs through sre_partial_sums (the same C-ABI call bench.py times) in chunks of
2^chunk_log2 X-strings; per-chunk device time from CUDA events; nvidia-smi samples the clocks.
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_07824_b200 as sre  # noqa: E402
import sre_inputs as si  # noqa: E402
from bench import Clocks, load_peaks  # noqa: E402

n = int(sys.argv[1])
kind = sys.argv[2]
chunk = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 19)
max_chunks = int(sys.argv[4]) if len(sys.argv) > 4 else None     # timing slices only (no pin)
alphas = [2.0]
t0 = time.time()
if kind == "scrambled":
    lo, hi = si.haar(n // 2, 24002), si.haar(n - n // 2, 24003)
    psi_h = si.scrambled_pair(lo, hi, 6, 24004)
else:
    psi_h = si.haar(n, 24001)
t_gen = time.time() - t0
psi = torch.from_numpy(psi_h).cuda()
ws = torch.empty(sre.workspace_size(n, 1, 1), dtype=torch.uint8, device="cuda")
out = torch.empty((1, 3), dtype=torch.float64, device="cuda")
sre.partial_sums(psi, 1 << 12, (1 << 12) + 64, alphas, out=out, workspace=ws)   # warm-up
torch.cuda.synchronize()
D = 1 << n
acc = np.zeros(3)
chunk_ms = []
clk = Clocks(0)
wall0 = time.perf_counter()
for a in range(0, D, chunk):
    if max_chunks is not None and len(chunk_ms) >= max_chunks:
        break
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sre.partial_sums(psi, a, min(D, a + chunk), alphas, out=out, workspace=ws)
    e1.record()
    e1.synchronize()
    chunk_ms.append(e0.elapsed_time(e1))
    acc += out.cpu().numpy()[0]          # fixed chunk order: deterministic
    print(f"# chunk {a // chunk + 1}/{(D + chunk - 1) // chunk}: {chunk_ms[-1]:.1f} ms", file=sys.stderr, flush=True)
wall = time.perf_counter() - wall0
clocks = clk.stop()
m, ln = sre.finalize(acc.reshape(1, 3), n, alphas)
dev_s = sum(chunk_ms) / 1e3
swept = min(D, len(chunk_ms) * chunk)
if swept < D:                                  # a timing slice: rates over the X-strings swept
    print(json.dumps({"N": n, "state": kind, "x_strings": swept, "device_seconds": dev_s,
                      "us_per_x_string": dev_s / swept * 1e6, "pauli_per_s": swept * 2.0 ** n / dev_s,
                      "frac_of_hbm": 16.0 * swept * 2.0 ** n / dev_s / 1e9 / load_peaks()[0]["hbm_gbs"],
                      "clocks": clocks}), flush=True)
    sys.exit(0)
peaks, psrc = load_peaks()
line = {
    "N": n, "state": kind, "alpha": alphas, "M2": float(m[0][0]), "lost_norm": float(ln[0]),
    "raw_sums": acc.tolist(), "device_seconds": dev_s, "wall_seconds": wall, "state_gen_seconds": t_gen,
    "pauli_per_s": 4.0 ** n / dev_s, "us_per_x_string": dev_s / D * 1e6,
    "fwht_hbm_GBps": 16.0 * 4.0 ** n / dev_s / 1e9,
    "frac_of_hbm": 16.0 * 4.0 ** n / dev_s / 1e9 / peaks["hbm_gbs"], "hbm_peak_GBps": peaks["hbm_gbs"],
    "hbm_peak_source": psrc, "chunks": len(chunk_ms), "chunk_x_strings": chunk,
    "chunk_ms_min": min(chunk_ms), "chunk_ms_max": max(chunk_ms), "clocks": clocks,
    "gpu": torch.cuda.get_device_name(0),
}
if kind == "scrambled":
    import oracle
    oracle.build()
    m_lo = oracle.sre(lo, alphas)[0][0]
    m_hi = oracle.sre(hi, alphas)[0][0]
    line.update({"pin": "M2(C(phi_hi x phi_lo)) = M2(phi_lo) + M2(phi_hi) (P:105-110)",
                 "M2_expected": m_lo + m_hi, "abs_err": abs(float(m[0][0]) - (m_lo + m_hi)),
                 "pass": abs(float(m[0][0]) - (m_lo + m_hi)) < 1e-10 and abs(float(ln[0])) < 1e-10})
else:
    target = math.log2(D + 3) - 2
    line.update({"sanity": "Haar M2 ~ log2(2^N + 3) - 2 within 40 2^-N (P:1155-1160)", "M2_haar_mean": target,
                 "pass": abs(float(m[0][0]) - target) < 40.0 / D and abs(float(ln[0])) < 1e-10})
print(json.dumps(line), flush=True)
