"""Spectrum epilogue throughput: python tools/spec_rate.py N [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07824_b200 as sre  # noqa: E402
import sre_inputs as si  # noqa: E402

n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
psi = torch.from_numpy(si.haar(n, 3)).cuda()
sre.spectrum(psi)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    h = sre.spectrum(psi)
dt = (time.perf_counter() - t0) / reps
print(f"N={n}: {dt * 1e3:.2f} ms per full spectrum, {4.0 ** n / dt:.3e} Pauli/s; top bins {h[:20].tolist()}")
