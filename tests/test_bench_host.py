"""Host-side pieces of bench.py / tools: roofline.traffic lookup and the ncu CSV reducer (no GPU)."""
import importlib.util
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _load(name, rel):
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, rel))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_ncu_traffic_reducer(tmp_path, monkeypatch):
    tool = _load("ncu_traffic", "tools/ncu_traffic.py")
    csv = tmp_path / "raw.csv"
    csv.write_text(
        '"Kernel Name","launch__grid_size","gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum"\n'
        '"","","us","Mbyte","Gbyte"\n'
        '"void k_legs<0, 4, 0, 256>(LegArgs)","296","400","100","1.5"\n'
        '"void k_legs<3, 2, 0>(LegArgs)","592","300","300","0.5"\n'
        '"void k_legs<3, 2, 1>(LegArgs)","740","200","700","0"\n')
    out = tmp_path / "t.json"
    monkeypatch.setattr(sys, "argv", ["x", str(out), f"x8:pass_a:{csv}:k_legs<\\d+, \\d+, 1"])
    tool.main()
    t = json.loads(out.read_text())["x8"]
    assert t["kind"] == "pass_a" and t["launches"] == 2
    assert abs(t["dram_bytes_per_launch"] - (1.6e9 + 0.8e9) / 2) < 1.0


def test_bench_traffic_lookup():
    bench = _load("bench_mod", "bench.py")
    assert bench.ncu_traffic("no-such-config", "pass_a") is None
    path = os.path.join(ROOT, "profiles", "r02_traffic.json")
    if os.path.exists(path):
        for cfg, t in json.load(open(path)).items():
            assert t["kind"] in ("pass_a", "pass_b", "single_pass")
            assert bench.ncu_traffic(cfg, t["kind"]) == t["dram_bytes_per_launch"] > 0
            other = "pass_b" if t["kind"] != "pass_b" else "pass_a"
            assert bench.ncu_traffic(cfg, other) is None


def test_roofline_accounting():
    """Algorithmic bytes/ops of the bench line: pass A = 8 B/Pauli + one psi read
    per launch, pass B = 8 B/Pauli, L = 10 (N <= 20) / 12 (N = 21..24) / 13 (N = 25); at N = 24 a pass A
    moving its bytes at exactly the HBM peak reads frac 1 (it cannot exceed 1 at any slower time)."""
    bench = _load("bench_mod", "bench.py")
    peaks = {"hbm_gbs": 6551.4}
    assert [bench.two_pass_L(n) for n in (15, 20, 21, 24, 25)] == [10, 10, 12, 12, 13]
    k = 32
    paulis = k * float(1 << 24)
    bytes_a = 8.0 * paulis + 16.0 * (1 << 24)
    t_ms = bytes_a / 6551.4e9 * 1e3
    r = bench.roofline(24, 1, [2.0], "pass_a", t_ms, paulis, peaks, "measured", 1965.0)
    assert r["bound"] == "hbm" and abs(r["frac"] - 1.0) < 1e-12
    assert abs(r["bytes_per_pauli"] - (8.0 + 16.0 / k)) < 1e-12
    assert r["fp64"]["ops_per_pauli"] == 2 + 12
    rb = bench.roofline(20, 1, [2.0], "pass_b", 1.0, 128 * float(1 << 20), peaks, "measured", 1965.0)
    assert rb["bytes_per_pauli"] == 8.0 and rb["fp64"]["ops_per_pauli"] == (20 - 1 - 10) + 3
    rs = bench.roofline(14, 256, [2.0], "single_pass", 1.0, 1e9, peaks, "measured", 1965.0)
    assert rs["bound"] == "alu" and rs["ops_per_pauli"] == 2 + 13 + 3
    # alpha in {1, 2, 3}: log (26) + t ln t FMA (1) + alpha 2 (2) + alpha 3 (3) on top of t and purity (2)
    assert bench.epilogue_ops([1.0, 2.0, 3.0]) == 2 + 26 + 1 + 2 + 3
    assert bench.epilogue_ops([2.0]) == 3
    assert bench.epilogue_ops([0.5]) == 2 + 26 + 22
