"""Small invocations of every kernel family, for compute-sanitizer (one tool per process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07824_b200 as sre  # noqa: E402
import sre_inputs as si  # noqa: E402

cases = [(3, 0, 8, [2.0]), (8, 0, 256, [1.0, 2.0, 3.0, 0.5, 1.5]), (12, 0, 4096, [2.0]), (14, 0, 64, [2.0]),
         (15, 0, 64, [2.0]), (16, 1024, 1024 + 40, [1.0, 2.0]), (20, 2048, 2048 + 24, [2.0]),
         (21, 4096, 4096 + 12, [2.0]), (21, 0, 3, [2.0])]
for n, lo, hi, al in cases:
    psi = torch.from_numpy(si.haar(n, 7 + n)).cuda()
    out = sre.partial_sums(psi, lo, hi, al)
    torch.cuda.synchronize()
    print(n, lo, hi, out.cpu().numpy().tolist()[0][:2], flush=True)
c = sre.chi(torch.from_numpy(si.haar(17, 3)).cuda(), 12345)
b = torch.from_numpy(si.haar_batch(10, 4, 5)).cuda()
print(sre.exact_batched(b, [2.0])[0].ravel().tolist())
print("done")
