"""bench.py output contract on a B200: one JSON line with every key the driver and DESIGN §9 rely on.

Runs the short configs (c3: 256 x N=14 states; x8: N_A=8 mixed mana) for one timed step; the
roofline must name a kernel that launched, and traffic must come from the committed ncu capture
when one exists for the config (profiles/r02_traffic.json)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "gpu_launches", "clocks", "e2e")


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c3", "x8"])
def test_bench_line_contract(config):
    d = _run("--config", config, "--steps", "1", "--warmup", "3", "--no-cpu-baseline")
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "alu", "tensor") and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert r["launches_timed"] > 0 and r["avg_launch_ms"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    path = os.path.join(ROOT, "profiles", "r02_traffic.json")
    t = json.load(open(path)).get(config) if os.path.exists(path) else None
    if t and t["kind"] == r["kernel"]:
        assert r["traffic"] == t["dram_bytes_per_launch"]
