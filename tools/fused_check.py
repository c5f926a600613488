"""Compare fused vs non-fused two-pass sums on full ranges (debug aid)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
code = r'''
import sys, time, torch, numpy as np
import paper_2601_07824_b200 as sre, sre_inputs as si
n=int(sys.argv[1]); lo=int(sys.argv[2]); hi=int(sys.argv[3])
psi=torch.from_numpy(si.haar(n, 99)).cuda()
torch.cuda.synchronize(); t0=time.time()
out=sre.partial_sums(psi, lo, hi, [2.0]); torch.cuda.synchronize()
print(repr(out.cpu().numpy().tolist()), time.time()-t0)
'''
for n, lo, hi in [(15, 0, 1 << 15), (16, 1024, 1024 + 4096), (17, 0, 1 << 17), (20, 1024, 1024 + 65536)]:
    r = {}
    for f in ("0", "1"):
        env = dict(os.environ, SRE_FUSED=f)
        p = subprocess.run([sys.executable, "-c", code, str(n), str(lo), str(hi)], env=env, capture_output=True, text=True, timeout=300)
        r[f] = (p.stdout.strip() or p.stderr[-500:])
    print(n, lo, hi, "nonfused:", r["0"], "\n          fused:   ", r["1"], flush=True)
