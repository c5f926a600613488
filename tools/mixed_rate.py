"""Throughput of the mixed-state mana path: python tools/mixed_rate.py N [reps]
Builds a product of single-qutrit mixtures on the device (9^N complex128), times the in-place
sre_mana_mixed_sums (refilled from a pristine copy before each call; the copy is not timed) and
prints elements/s, HBM GB/s of the passes and the per-pass launch times."""
import json
import sys

import torch

import paper_2601_07824_b200 as sre
from paper_2601_07824_b200 import qutrit
import sre_inputs.qutrit as q

n = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rho = torch.ones((1, 1), dtype=torch.complex128, device="cuda")
for k in range(n):
    rho = torch.kron(torch.from_numpy(q.mixed_strange(0.3 + 0.07 * k)).cuda(), rho)
flat0 = rho.t().contiguous().view(-1)
del rho
out = torch.empty(2, dtype=torch.float64, device="cuda")
times = []
if n >= 10:   # no room for a pristine copy: the first call gives the sums; later in-place calls
    work = flat0  # run on the transformed buffer (same work, same time; their sums are meaningless)
    qutrit.mixed_sums_(work, n, out=out)
    first = out.cpu().tolist()
else:
    work = torch.empty_like(flat0)
    work.copy_(flat0)
    qutrit.mixed_sums_(work, n, out=out)
sre.profile_begin(1)
for r in range(reps):
    if work is not flat0:
        work.copy_(flat0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    qutrit.mixed_sums_(work, n, out=out)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
prof = sre.profile_end()
ms = sum(times) / len(times)
el = 9.0 ** n
print(json.dumps({"N": n, "ms": ms, "elements_per_s": el / (ms * 1e-3),
                  "sums": first if n >= 10 else out.cpu().tolist(),
                  "prof": {k: v for k, v in prof.items() if v["launched"]}}))
