"""Per-call latency of sre_x_string_sums (the sampler's energy batch): python tools/xs_rate.py N n_a [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_07824_b200 as sre  # noqa: E402
import sre_inputs as si  # noqa: E402

n, na = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 200
psi = torch.from_numpy(si.haar(n, 5)).cuda()
ws = torch.empty(sre.workspace_size(n, 1, 1), dtype=torch.uint8, device="cuda")
rng = np.random.default_rng(0)
a = rng.integers(0, 1 << n, size=na, dtype=np.uint64)
out = sre.x_string_sums(psi, a, [2.0], workspace=ws)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    out = sre.x_string_sums(psi, a, [2.0], workspace=ws)
    s = out[:, 0].cpu().numpy()          # the sampler reads the energies back every step
dt = (time.perf_counter() - t0) / reps
print(f"N={n} n_a={na}: {dt * 1e6:.1f} us per call (incl. D2H), {na / dt:.3e} energies/s")
