"""Throughput of the mana path: python tools/mana_rate.py N count [reps]
Times sre_mana_partial_sums over X-strings [0, count) with CUDA events; prints phase-space
points / s (count * 3^N per call) and the per-kind launch times."""
import json
import sys

import torch

import paper_2601_07824_b200 as sre
from paper_2601_07824_b200 import qutrit
import sre_inputs.qutrit as q

n = int(sys.argv[1])
count = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
psi = torch.from_numpy(q.haar(n, 42)).cuda()
ws = torch.empty(qutrit.workspace_size(n), dtype=torch.uint8, device="cuda")
out = torch.empty(2, dtype=torch.float64, device="cuda")
qutrit.partial_sums(psi, 0, count, out=out, workspace=ws)
torch.cuda.synchronize()
sre.profile_begin(1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    qutrit.partial_sums(psi, 0, count, out=out, workspace=ws)
e1.record()
torch.cuda.synchronize()
prof = sre.profile_end()
ms = e0.elapsed_time(e1) / reps
pts = count * 3 ** n
print(json.dumps({"N": n, "count": count, "ms": ms, "points_per_s": pts / (ms * 1e-3),
                  "us_per_xstring": ms * 1e3 / count, "prof": prof}))
