"""Throughput of partial_sums on a slice: python tools/rate.py N a0 count [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07824_b200 as sre  # noqa: E402
import sre_inputs as si  # noqa: E402

n, a0, cnt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
prec = sys.argv[5] if len(sys.argv) > 5 else "fp64"
alphas = [float(x) for x in sys.argv[6].split(",")] if len(sys.argv) > 6 else [2.0]
psi = torch.from_numpy(si.haar(n, 1234)).cuda()
ws = torch.empty(sre.workspace_size(n, 1, len(alphas), prec), dtype=torch.uint8, device="cuda")
out = sre.partial_sums(psi, a0, a0 + cnt, alphas, workspace=ws, precision=prec)
torch.cuda.synchronize()
sre.profile_begin(1)
t0 = time.perf_counter()
for _ in range(reps):
    out = sre.partial_sums(psi, a0, a0 + cnt, alphas, workspace=ws, precision=prec)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
prof = sre.profile_end()
print(f"{prec} N={n} count={cnt}: {dt*1e3:.2f} ms, {cnt * 2.0**n / dt:.3e} Pauli/s, per X-string {dt/cnt*1e6:.2f} us",
      {k: (round(v['ms_sum'] / max(1, v['timed']), 4), v['launched']) for k, v in prof.items() if v['launched']})
