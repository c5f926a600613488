"""Freeze full-size oracle values as JSON fixtures (calls only oracle/ and sre_inputs/).

    python tools/make_fixtures.py c2      # N=16 Haar seed 16001, alpha in {1,2,3}   (minutes)
    python tools/make_fixtures.py c4      # N=20 Haar seed 20001, alpha = 2  (~15 h on 8 cores: not frozen)

Each fixture records the input recipe and the SHA-256 of the state's bytes, so a test can
regenerate the identical state and compare the CUDA path with the frozen oracle sums.
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import sre_inputs as si  # noqa: E402

CASES = {
    "c2": dict(n=16, seed=16001, alphas=[1.0, 2.0, 3.0]),
    "c4": dict(n=20, seed=20001, alphas=[2.0]),
}


def main(name):
    c = CASES[name]
    psi = si.haar(c["n"], c["seed"])
    sha = hashlib.sha256(psi.tobytes()).hexdigest()
    t0 = time.time()
    sums = oracle.sums_fwht(psi, c["alphas"])
    wall = time.time() - t0
    m, ln = oracle.finalize(sums, c["n"], c["alphas"])
    out = dict(
        config=name, generator="sre_inputs.haar", n=c["n"], seed=c["seed"], alphas=c["alphas"],
        psi_sha256=sha, oracle_mode="fwht (Alg. 2, long double)", sums=[float(x) for x in sums],
        M=m, lost_norm=ln, oracle_wall_s=wall, oracle_threads=oracle.num_threads(),
        source="written by tools/make_fixtures.py; values come from oracle/ only",
    )
    path = os.path.join(ROOT, "tests", "golden", f"oracle_{name}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, m, ln, wall)


if __name__ == "__main__":
    main(sys.argv[1])
