"""Short driver for ncu: partial sums of a slice of X-strings of a seeded Haar state.
    python tools/prof_range.py N a_begin count [alpha ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07824_b200 as sre  # noqa: E402
import sre_inputs as si  # noqa: E402

n, a0, cnt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
alphas = [float(x) for x in sys.argv[4:]] or [2.0]
psi = torch.from_numpy(si.haar(n, 20001 if n == 20 else 1234)).cuda()
out = sre.partial_sums(psi, a0, a0 + cnt, alphas)
torch.cuda.synchronize()
print(out.cpu().numpy())
