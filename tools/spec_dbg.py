"""Debug: |T>^n spectrum from the library vs the oracle's closed form, printing differing bins."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2601_07824_b200 as sre  # noqa: E402
import sre_inputs as si  # noqa: E402

n = int(sys.argv[1])
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 1 << n
psi = torch.from_numpy(si.t_state(n)).cuda()
g = sre.spectrum(psi, lo, hi)
if lo == 0 and hi == 1 << n:
    o = oracle.t_state_spectrum(n)
else:
    o = oracle.spectrum(si.t_state(n), (lo, hi))
d = np.nonzero(g != o)[0]
print(f"N={n} [{lo},{hi}) mismatched bins {d.tolist()}: gpu {g[d].tolist()} oracle {o[d].tolist()}")
