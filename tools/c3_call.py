"""One bench-equivalent call of config 3 (256 x N = 14 Clifford+T states, alpha = 2) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07824_b200 as sre  # noqa: E402
import sre_inputs as si  # noqa: E402

batch, _ = si.config3_batch(14, 256, 14000)
t = torch.from_numpy(batch).cuda()
out = sre.partial_sums(t, 0, 1 << 14, [2.0])
torch.cuda.synchronize()
print(out[:2].cpu().numpy())
