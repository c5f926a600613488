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
    path = os.path.join(ROOT, "profiles", "r01_traffic.json")
    if os.path.exists(path):
        for cfg, t in json.load(open(path)).items():
            assert t["kind"] in ("pass_a", "pass_b", "single_pass")
            assert bench.ncu_traffic(cfg, t["kind"]) == t["dram_bytes_per_launch"] > 0
            other = "pass_b" if t["kind"] != "pass_b" else "pass_a"
            assert bench.ncu_traffic(cfg, other) is None
