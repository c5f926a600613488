#!/usr/bin/env python
"""Benchmark of the exact-SRE hot path (BASELINE.json metric: exact SRE M_2 Pauli strings/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4|c2|c3|c5] [--impl reference]

A step = one full evaluation of Alg. 2 for the config's workload: every
X-string's generation + Walsh-Hadamard transform + FP64 power sums, the reduction, the
cross-GPU allreduce (N > 1) and the host finalisation of Eq. (2).  Default workload: BASELINE
config 4 (N = 20 seeded Haar state, alpha = 2), 4^20 Pauli strings per step.  Under torchrun the
2^N X-strings are split into contiguous equal shards, one per rank, and the (n_alpha + 2) partial
sums are combined with one NCCL all_reduce per step (strong scaling: total work fixed).

``--impl reference`` times the CPU oracle (oracle/, plain C, long double) on the host cores on a
bounded sample of the same workload (the only reference this paper-only task has).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "exact SRE M_2 Pauli strings/s at N=20/24 on 1-8 B200; FWHT HBM GB/s vs peak"
CONFIGS = {
    # name: (workload label, N, batch, alphas, seed)
    "c4": ("N=20 seeded Haar state, alpha=2 (BASELINE config 4)", 20, 1, [2.0], 20001),
    "c2": ("N=16 seeded Haar state, alpha in {1,2,3} (BASELINE config 2)", 16, 1, [1.0, 2.0, 3.0], 16001),
    "c3": ("256 x N=14 Clifford+T states, alpha=2 (BASELINE config 3)", 14, 256, [2.0], 14000),
    "c5": ("N=24 seeded Haar state, alpha=2 (BASELINE config 5)", 24, 1, [2.0], 24001),
}
# Pure-state qutrit mana (NEXT-3, Alg. 5): name -> (workload label, N qutrits, brick-wall depth, seed)
MANA_CONFIGS = {
    "m12": ("N=12 qutrit brick-wall state, depth 4 (pure-state mana, PAPER Table II row N=12, P:1449-1466)", 12, 4, 12012),
    "m14": ("N=14 qutrit brick-wall state, depth 4 (pure-state mana, PAPER Table II row N=14, P:1449-1466)", 14, 4, 14014),
}
MANA_METRIC = "exact pure-state qutrit mana, phase-space points/s (9^N per state)"
# Mixed-state qutrit mana (NEXT-4, Alg. 6): name -> (label, N_A kept qutrits, N total, depth, seed)
MIXED_CONFIGS = {
    "x8": ("rho_A of an N=10 qutrit brick-wall state (depth 3) on N_A=8 qutrits (PAPER P:1418-1430, Table II N_A=8)",
           8, 10, 3, 10003),
    "x10": ("rho_A of an N=12 qutrit brick-wall state (depth 4) on N_A=10 qutrits (PAPER Table II N_A=10, 56 GB)",
            10, 12, 4, 12004),
}
MIXED_METRIC = "exact mixed-state qutrit mana, phase-space points/s (9^N_A per density matrix)"
FP64_OPS_PER_CLK_SM = 64        # B200 FP64 pipe (measured 63.9/clk/SM, profiles/r01_microbench.json)


def ncu_traffic(config, kind):
    """roofline.traffic: DRAM bytes per launch of the dominant kernel from the committed `ncu --set full`
    capture of this config (profiles/r02_traffic.json, written by tools/ncu_traffic.py), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_traffic.json")) as f:
            t = json.load(f).get(config)
    except (OSError, ValueError):
        return None
    return t["dram_bytes_per_launch"] if t and t.get("kind") == kind else None


def two_pass_L(n):
    """Low-bit count of pass A per N (csrc/sre_api.cu two_pass_params)."""
    if n <= 20:
        return 10
    return 12 if n <= 24 else 13


def epilogue_ops(alphas):
    """FP64 ops per Pauli string of the power-sum epilogue: t = y^2 and the purity
    add (2); alpha = 2 alone: 1 FMA; integer alpha: (alpha - 1) multiplies + 1 add; alpha = 1: the
    logarithm (ln_fast: 9-term polynomial + division + scaling, ~26) + 1 FMA; non-integer alpha:
    the shared logarithm + exp_fast (~20) + 2."""
    ops = 2
    if alphas == [2.0]:
        return ops + 1
    need_log = any(a == 1.0 for a in alphas)
    real = [a for a in alphas if not (a == int(a) and 1 <= a <= 64)]
    if need_log or real:
        ops += 26
    if need_log:
        ops += 1
    for a in alphas:
        if a == 1.0:
            continue
        ops += (int(a) - 1 + 1) if a == int(a) else 22
    return ops


def roofline(n, b, alphas, dom, avg_ms, paulis_per_launch, peaks, peak_src, sm_mhz):
    """roofline object of the bench line for the dominant kernel kind.
    Two-pass N >= 15: HBM-bound -- pass A moves 8 B/Pauli of workspace writes plus one read of psi per
    launch (2^N x 16 B: the launch's X-strings re-read each psi row from L2); pass B reads 8 B/Pauli.
    Single pass N <= 14: no workspace; FP64-pipe bound (psi operands from L2).  Alongside: the FP64
    fraction of the same kernel at the run's max SM clock."""
    fp64_peak = FP64_OPS_PER_CLK_SM * 148 * sm_mhz * 1e6 / 1e12
    L = two_pass_L(n)
    if dom == "pass_a":
        ops = 2 + L
        bytes_launch = 8.0 * paulis_per_launch + 16.0 * (1 << n) * b
    elif dom == "pass_b":
        ops = (n - 1 - L) + epilogue_ops(alphas)
        bytes_launch = 8.0 * paulis_per_launch
    else:
        ops = 2 + (n - 1) + epilogue_ops(alphas)
        bytes_launch = None
    fp64 = ops * paulis_per_launch / (avg_ms * 1e-3) / 1e12
    fp64_obj = {"achieved": fp64, "peak": fp64_peak, "unit": "TFLOP/s (FP64 ops)", "frac": fp64 / fp64_peak,
                "ops_per_pauli": ops,
                "peak_source": f"64 FP64 ops/clk/SM x 148 SMs x {sm_mhz:.0f} MHz (guide unit count; measured 63.9)"}
    if bytes_launch is not None:
        gbs = bytes_launch / (avg_ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": gbs / peaks["hbm_gbs"], "traffic": None, "peak_source": peak_src,
                "bytes_per_launch": bytes_launch, "bytes_per_pauli": bytes_launch / paulis_per_launch,
                "fp64": fp64_obj}
    return {"bound": "alu", "achieved": fp64, "peak": fp64_peak, "unit": "TFLOP/s (FP64 ops)",
            "frac": fp64 / fp64_peak, "traffic": None, "peak_source": fp64_obj["peak_source"], "ops_per_pauli": ops}


def ncu_limiter(config, kind):
    """The measured limiter of the dominant kernel from its committed `ncu --set full` capture
    (profiles/r02_limiters.json, written from the summaries in profiles/), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_limiters.json")) as f:
            t = json.load(f).get(config, {}).get(kind)
    except (OSError, ValueError):
        return None
    return t


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def make_state(cfg):
    import sre_inputs as si
    _, n, b, _, seed = CONFIGS[cfg]
    if cfg == "c3":
        batch, _ = si.config3_batch(n, b, seed)
        return batch
    return si.haar(n, seed)


class Clocks:
    """nvidia-smi sampler running during the timed region (the recipe's clocks line)."""

    def __init__(self, gpu_index):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        self.t0 = time.time()

    def stop(self, min_seconds=0.5):
        if self.p is None:
            return None
        if time.time() - self.t0 < min_seconds:      # short timed regions: let nvidia-smi take a sample
            time.sleep(min_seconds - (time.time() - self.t0))
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows]
        mx = float(rows[0][2])
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].strip().lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows), "power_w_max": max(float(r[3]) for r in rows)}


def cpu_sample(cfg, seconds_target=15.0):
    """Oracle (Alg. 2, long double, OpenMP) on a bounded slice of the workload's X-strings."""
    import oracle
    label, n, b, alphas, seed = CONFIGS[cfg]
    psi = make_state(cfg)
    one = psi[0] if b > 1 else psi
    # calibrate the slice: X-strings cost N 2^N each, uniform
    threads = oracle.num_threads()
    k = max(threads, 1)
    t0 = time.perf_counter()
    oracle.sums_fwht(one, alphas, a_range=(0, k))
    dt = time.perf_counter() - t0
    per_a = dt / k
    k2 = int(min(1 << n, max(threads, seconds_target / max(per_a, 1e-9))))
    k2 = max(threads, (k2 // threads) * threads)
    t0 = time.perf_counter()
    oracle.sums_fwht(one, alphas, a_range=(0, k2))
    dt = time.perf_counter() - t0
    paulis = k2 * float(1 << n)
    return {"value": paulis / dt, "unit": "Pauli strings/s", "cores": threads, "kind": "oracle",
            "sample": f"oracle fwht (Alg. 2, long double) over X-strings [0, {k2}) of the {label}; "
                      f"{k2} x 2^{n} Pauli strings in {dt:.2f} s", "seconds": dt}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = args.config
    label, n, b, alphas, seed = CONFIGS[cfg]
    import oracle
    oracle.build()
    psi = make_state(cfg)
    one = psi[0] if b > 1 else psi
    threads = oracle.num_threads()
    # each step: a bounded slice sized so the whole run stays within a few minutes
    k = max(threads, 1)
    t0 = time.perf_counter()
    oracle.sums_fwht(one, alphas, a_range=(0, k))
    per_a = (time.perf_counter() - t0) / k
    budget = 150.0 / max(1, args.steps + args.warmup)
    ka = int(max(threads, min(1 << n, budget / max(per_a, 1e-9))))
    ka = max(threads, (ka // threads) * threads)
    for _ in range(args.warmup):
        oracle.sums_fwht(one, alphas, a_range=(0, ka))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.sums_fwht(one, alphas, a_range=(0, ka))
        times.append(time.perf_counter() - t0)
    dt = sum(times)
    value = args.steps * ka * float(1 << n) / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Pauli strings/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (long double accum)",
        "data": "synthetic", "config": {"workload": label, "N": n, "batch": b, "alphas": alphas, "seed": seed,
                                        "x_strings_per_step": ka},
        "cpu_baseline": {"value": value, "unit": "Pauli strings/s", "cores": threads, "kind": "oracle",
                         "sample": f"oracle fwht over X-strings [0, {ka}) per step ({ka} of 2^{n})"},
        "e2e": {"value": value, "unit": "Pauli strings/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def mana_state(cfg):
    import sre_inputs.qutrit as q
    _, n, depth, seed = MANA_CONFIGS[cfg]
    return q.brickwall(n, depth, seed)


def mana_cpu_sample(psi, n, label, seconds_target):
    """Oracle (Alg. 5, long double, OpenMP) over a bounded slice [0, k) of the X-strings."""
    import oracle
    from oracle import mana as om
    threads = oracle.num_threads()
    k = max(threads, 1)
    t0 = time.perf_counter()
    om.sums_fwht(psi, (0, k))
    per_a = (time.perf_counter() - t0) / k
    k2 = int(min(3 ** n, max(threads, seconds_target / max(per_a, 1e-9))))
    k2 = max(threads, (k2 // threads) * threads)
    t0 = time.perf_counter()
    om.sums_fwht(psi, (0, k2))
    dt = time.perf_counter() - t0
    return {"value": k2 * float(3 ** n) / dt, "unit": "phase-space points/s", "cores": threads, "kind": "oracle",
            "sample": f"oracle mana fwht (Alg. 5, long double) over X-strings [0, {k2}) of the {label}; "
                      f"{k2} x 3^{n} points in {dt:.2f} s", "seconds": dt}, k2


def run_mana_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    label, n, depth, seed = MANA_CONFIGS[args.config]
    import oracle
    oracle.build()
    psi = mana_state(args.config)
    budget = 150.0 / max(1, args.steps + args.warmup)
    cb, k = mana_cpu_sample(psi, n, label, budget)
    from oracle import mana as om
    for _ in range(args.warmup):
        om.sums_fwht(psi, (0, k))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        om.sums_fwht(psi, (0, k))
        times.append(time.perf_counter() - t0)
    dt = sum(times)
    value = args.steps * k * float(3 ** n) / dt
    cb.update({"value": value, "sample": f"oracle mana fwht over X-strings [0, {k}) per step ({k} of 3^{n})"})
    print(json.dumps({
        "impl": "reference", "metric": MANA_METRIC, "value": value, "unit": "phase-space points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (long double accum)",
        "data": "synthetic", "config": {"workload": label, "N": n, "depth": depth, "seed": seed,
                                        "x_strings_per_step": k},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "phase-space points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


def main_mana(args):
    """A step = the full Alg. 5 sweep of one N-qutrit state (all 3^N X-strings, 9^N phase-space
    points), sharded over ranks by contiguous X-string ranges, one all_reduce of 2 doubles, and the
    host log2 of Eq. (10)."""
    import math

    import torch
    import torch.distributed as dist

    import paper_2601_07824_b200 as sre
    from paper_2601_07824_b200 import qutrit

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    label, n, depth, seed = MANA_CONFIGS[args.config]
    na = 3 ** n
    from paper_2601_07824_b200.dist import shard_bounds
    lo, hi = shard_bounds(na, rank, world)              # contiguous X-string shard
    psi_host = mana_state(args.config)
    psi = torch.from_numpy(psi_host).to(dev)
    ws = torch.empty(qutrit.workspace_size(n), dtype=torch.uint8, device=dev)
    sums = torch.empty(2, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        qutrit.partial_sums(psi, lo, hi, out=sums, workspace=ws, stream=stream)
        if world > 1:
            dist.all_reduce(sums)
        h = sums.cpu().numpy()
        return math.log2(h[0] / na), h[1] / na

    for _ in range(max(args.warmup, 0)):
        m, n2 = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    launches0 = sre.launch_count()
    sre.profile_begin(max(1, args.profile_stride // 4))
    step_ms = []
    for _ in range(args.steps):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        m, n2 = step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    prof = sre.profile_end()
    launches = sre.launch_count() - launches0
    clk = clocks.stop()
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        dist.barrier()
    pts = 9.0 ** n
    value = args.steps * pts / (tot_ms * 1e-3)
    e2e = None
    if world == 1:
        pinned = torch.from_numpy(psi_host).pin_memory()
        t_e = []
        for _ in range(max(1, min(args.steps, 2))):
            t0 = time.perf_counter()
            qutrit.mana(pinned)                               # H2D + sweep + D2H of the 2 sums
            t_e.append(time.perf_counter() - t0)
        e2e = {"value": pts * len(t_e) / sum(t_e), "unit": "phase-space points/s",
               "h2d_bytes_per_step": int(psi_host.nbytes), "d2h_bytes_per_step": 16,
               "ms_per_step": 1e3 * sum(t_e) / len(t_e)}
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    peaks, _ = load_peaks()
    kinds = {k: v for k, v in prof.items() if v["timed"] > 0 and k != "aux"}
    share = {k: v["ms_sum"] / v["timed"] * v["launched"] for k, v in kinds.items()}
    dom = max(share, key=share.get)
    avg_ms = prof[dom]["ms_sum"] / prof[dom]["timed"]
    pts_per_launch = pts * args.steps / max(1, world) / prof[dom]["launched"]
    # FP64 ops per phase-space point: pass A = gen 5 + 2 L, pass B = 2 H + 2
    L = {9: 5, 10: 6, 11: 6, 12: 7, 13: 7, 14: 7, 15: 8, 16: 8}.get(n, n)
    ops_pt = {"pass_a": 5 + 2 * L, "pass_b": 2 * (n - L) + 2, "single_pass": 5 + 2 * n + 2}[dom]
    sm_mhz = (clk or {}).get("sm_max_mhz", peaks.get("sm_max_mhz", 1965.0))
    peak = FP64_OPS_PER_CLK_SM * 148 * sm_mhz * 1e6 / 1e12
    achieved = ops_pt * pts_per_launch / (avg_ms * 1e-3) / 1e12
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s (FP64 ops)", "frac": achieved / peak,
            "traffic": ncu_traffic(args.config, dom), "kernel": dom, "avg_launch_ms": avg_ms, "launches_timed": prof[dom]["timed"],
            "share_of_step": share[dom] / tot_ms if world == 1 else None, "ops_per_point": ops_pt,
            "peak_source": f"64 FP64 ops/clk/SM x 148 SMs x {sm_mhz:.0f} MHz",
            "note": "measured limiter is the L1TEX/shared-memory data pipe (profiles/r01_ncu_summary_mana14.txt)"}
    line = {
        "metric": MANA_METRIC, "value": value, "unit": "phase-space points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": label, "N": n, "depth": depth, "seed": seed, "x_string_shards": world,
                   "l2": "flushed between steps (256 MiB write)",
                   "step": "mana partial sums over all 3^N X-strings + allreduce + log2"},
        "roofline": roof, "gpu_launches": int(launches), "clocks": clk, "e2e": e2e,
        "result": {"mana": m, "norm2": n2}, "profile": prof,
    }
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        line["cpu_baseline"], _ = mana_cpu_sample(psi_host, n, label, 15.0)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def mixed_phi(cfg):
    """Phi[x_B, x_A] of the config's pure state (rho_A = Phi^T conj(Phi), qutrits 0..N_A-1 kept)."""
    import sre_inputs.qutrit as q
    _, na, n, depth, seed = MIXED_CONFIGS[cfg]
    return q.brickwall(n, depth, seed).reshape(3 ** (n - na), 3 ** na)


def mixed_oracle_sample(seconds_hint=None):
    """Oracle Alg. 6 (long double, OpenMP over fibers) on the x8 workload: the full transform is
    not divisible into independent units, so the bounded sample is the whole N_A = 8 problem."""
    import oracle
    from oracle import mana as om
    phi = mixed_phi("x8")
    rho = phi.T @ np.conj(phi)
    t0 = time.perf_counter()
    om.sums_mixed_alg6(rho)
    dt = time.perf_counter() - t0
    return {"value": 9.0 ** 8 / dt, "unit": "phase-space points/s", "cores": oracle.num_threads(), "kind": "oracle",
            "sample": f"oracle Alg. 6 (long double, dense 9x9 leg sweep) on the full x8 problem "
                      f"(N_A=8, 9^8 points) in {dt:.2f} s", "seconds": dt}


def run_mixed_reference(args):
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    label, na, n, depth, seed = MIXED_CONFIGS[args.config]
    import oracle
    oracle.build()
    times = []
    for i in range(args.warmup + args.steps):
        cb = mixed_oracle_sample()
        if i >= args.warmup:
            times.append(cb["seconds"])
    dt = sum(times)
    value = args.steps * 9.0 ** 8 / dt
    cb.update({"value": value})
    print(json.dumps({
        "impl": "reference", "metric": MIXED_METRIC, "value": value, "unit": "phase-space points/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64 (long double accum)",
        "data": "synthetic", "config": {"workload": label, "N_A": na, "N": n, "depth": depth, "seed": seed,
                                        "oracle_problem": "x8 (N_A=8) -- the whole transform is the smallest unit"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "phase-space points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


def main_mixed(args):
    """A step = Alg. 6 on one density matrix: the full leg sweep M^{(x)N_A} in place on the
    column-major rho (fused multi-leg passes), the sums, and the host log2.  The input is
    regenerated on the device (rho_A = Phi^H Phi, cuBLAS) before each step, outside the timed
    region (the in-place transform consumes it).  Single GPU: the sweep has no X-string loop to
    shard (replicas only)."""
    import math

    import torch

    import paper_2601_07824_b200 as sre
    from paper_2601_07824_b200 import qutrit

    import torch.distributed as dist

    local = int(os.environ.get("LOCAL_RANK", "0"))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:                                   # replicas: no data-path collective, timing only
        dist.init_process_group("nccl", device_id=dev)
    label, na, n, depth, seed = MIXED_CONFIGS[args.config]
    d = 3 ** na
    phi = torch.from_numpy(mixed_phi(args.config)).to(dev)
    flat = torch.empty(d * d, dtype=torch.complex128, device=dev)
    out = torch.empty(2, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def regen():                                   # column-major rho: X[c, r] = rho[r, c] = (Phi^H Phi)[c, r]
        torch.matmul(phi.conj().t(), phi, out=flat.view(d, d))

    def step():
        qutrit.mixed_sums_(flat, na, out=out, stream=stream)
        h = out.cpu().numpy()
        return math.log2(h[0] / d), h[1] / d

    for _ in range(max(args.warmup, 0)):
        regen()
        m, tr = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    launches0 = sre.launch_count()
    sre.profile_begin(1)
    step_ms = []
    for _ in range(args.steps):
        regen()                                    # > L2: the 9^N_A x 16 B input itself flushes L2
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        m, tr = step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    prof = sre.profile_end()
    launches = sre.launch_count() - launches0
    clk = clocks.stop()
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
    pts = 9.0 ** na
    value = world * args.steps * pts / (tot_ms * 1e-3)   # every replica processes the whole rho
    # e2e: sre_mana_mixed from pinned host memory (H2D of the whole rho inside the timed region)
    e2e = None
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    nbytes = d * d * 16
    if world == 1 and avail > 2.5 * nbytes:
        regen()
        host = torch.empty(d * d, dtype=torch.complex128, pin_memory=True)
        host.copy_(flat)
        del flat
        torch.cuda.empty_cache()
        t_e = []
        for _ in range(2 if na <= 8 else 1):
            t0 = time.perf_counter()
            qutrit.mana_mixed(host)               # 1-D column-major flat: H2D + sweep + D2H
            t_e.append(time.perf_counter() - t0)
        e2e = {"value": pts * len(t_e) / sum(t_e), "unit": "phase-space points/s", "h2d_bytes_per_step": nbytes,
               "d2h_bytes_per_step": 16, "ms_per_step": 1e3 * sum(t_e) / len(t_e)}
    else:
        e2e = {"value": None, "unit": "phase-space points/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": 16,
               "note": f"host has {avail / 2**30:.0f} GiB available, < 2.5 x {nbytes / 2**30:.0f} GiB needed"}
    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0
    peaks, psrc = load_peaks()
    kinds = {k: v for k, v in prof.items() if v["timed"] > 0 and k != "aux"}
    share = {k: v["ms_sum"] / v["timed"] * v["launched"] for k, v in kinds.items()}
    dom = max(share, key=share.get)
    avg_ms = prof[dom]["ms_sum"] / prof[dom]["timed"]
    bytes_launch = (2.0 if dom == "pass_a" else 1.0) * nbytes    # non-final pass: read + write; final: read
    achieved = bytes_launch / (avg_ms * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": ncu_traffic(args.config, dom), "kernel": dom, "avg_launch_ms": avg_ms,
            "launches_timed": prof[dom]["timed"], "share_of_step": share[dom] / tot_ms,
            "bytes_per_launch": bytes_launch, "peak_source": psrc}
    line = {
        "metric": MIXED_METRIC, "value": value, "unit": "phase-space points/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": label, "N_A": na, "N": n, "depth": depth, "seed": seed,
                   "l2": f"input ({nbytes / 2**20:.0f} MiB) larger than L2, regenerated before each step (untimed)",
                   "step": "in-place fused leg sweep + sums + log2", "parallelism": "replicas only"},
        "roofline": roof, "gpu_launches": int(launches), "clocks": clk, "e2e": e2e,
        "result": {"mana": m, "trace": tr}, "profile": prof,
    }
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        line["cpu_baseline"] = mixed_oracle_sample()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS) + sorted(MANA_CONFIGS) + sorted(MIXED_CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-stride", type=int, default=16)
    args = ap.parse_args()
    if args.config in MANA_CONFIGS:
        return run_mana_reference(args) if args.impl == "reference" else main_mana(args)
    if args.config in MIXED_CONFIGS:
        return run_mixed_reference(args) if args.impl == "reference" else main_mixed(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2601_07824_b200 as sre

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    label, n, b, alphas, seed = CONFIGS[args.config]
    D = 1 << n
    from paper_2601_07824_b200.dist import shard_range, state_shard
    by_state = b > 1 and b >= world and world > 1      # batched workload: whole states per rank
    lo, hi = (0, D) if by_state else shard_range(n, rank, world)   # else a contiguous X-string shard
    s0, s1 = state_shard(b, rank, world) if by_state else (0, b)
    psi_host = make_state(args.config)
    psi = torch.from_numpy(psi_host).to(dev)            # replicated on every GPU (same seed)
    ws = torch.empty(sre.workspace_size(n, b, len(alphas)), dtype=torch.uint8, device=dev)
    sums = torch.zeros((b, len(alphas) + 2), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > L2 (126 MB)
    stream = torch.cuda.current_stream(dev)
    mine = psi[s0:s1] if b > 1 else psi

    def step():
        if s1 > s0:
            sre.partial_sums(mine, lo, hi, alphas, out=sums[s0:s1], workspace=ws, stream=stream)
        if world > 1:
            dist.all_reduce(sums)                        # the one exchange step (NCCL, NVLink)
        return sre.finalize(sums, n, alphas)             # D2H of (n_alpha+2) doubles per state

    for _ in range(max(args.warmup, 0)):
        m, ln = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local) if rank == 0 or True else None
    launches0 = sre.launch_count()
    sre.profile_begin(args.profile_stride)
    step_ms = []
    for _ in range(args.steps):
        flush.fill_(1)                                   # L2 flush between timed steps (untimed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        m, ln = step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
    prof = sre.profile_end()
    launches = sre.launch_count() - launches0
    torch.cuda.synchronize()
    clk = clocks.stop() if clocks else None
    tot_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        dist.barrier()
    paulis_per_step = float(b) * 4.0 ** n
    value = args.steps * paulis_per_step / (tot_ms * 1e-3)
    rank_paulis_per_step = float(s1 - s0) * 4.0 ** n * (hi - lo) / D   # this rank's share

    # ---- end-to-end through the public C entry with host (pinned) buffers, N=1 semantics per rank
    e2e = None
    if world == 1:
        pinned = torch.from_numpy(psi_host).pin_memory()
        fn = sre.exact if b == 1 else sre.exact_batched
        fn(pinned, alphas)
        torch.cuda.synchronize()
        t_e = []
        for _ in range(max(1, min(args.steps, 3))):
            t0 = time.perf_counter()
            fn(pinned, alphas)                             # H2D copy + norm check + sweep + D2H inside
            t_e.append(time.perf_counter() - t0)
        e2e = {"value": paulis_per_step * len(t_e) / sum(t_e), "unit": "Pauli strings/s",
               "h2d_bytes_per_step": int(psi_host.nbytes), "d2h_bytes_per_step": int(8 * b * (len(alphas) + 2)),
               "ms_per_step": 1e3 * sum(t_e) / len(t_e)}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    peaks, peak_src = load_peaks()
    kinds = {k: v for k, v in prof.items() if v["timed"] > 0 and k != "aux"}
    share = {k: v["ms_sum"] / v["timed"] * v["launched"] for k, v in kinds.items()}
    dom = max(share, key=share.get)
    avg_ms = prof[dom]["ms_sum"] / prof[dom]["timed"]
    launched = prof[dom]["launched"]
    paulis_per_launch = rank_paulis_per_step * args.steps / launched
    sm_mhz = (clk or {}).get("sm_max_mhz", peaks.get("sm_max_mhz", 1965.0))
    roof = roofline(n, b, alphas, dom, avg_ms, paulis_per_launch, peaks, peak_src, sm_mhz)
    roof["traffic"] = ncu_traffic(args.config, dom)
    roof.update({"kernel": dom, "avg_launch_ms": avg_ms, "launches_timed": prof[dom]["timed"],
                 "share_of_step": share[dom] / tot_ms if world == 1 else None})
    lim = ncu_limiter(args.config, dom)
    if lim:
        roof["limiter"] = lim
    hbm_equiv = 16.0 * value / max(1, world) / 1e9      # FWHT workspace bytes per Pauli string (16 B)
    line = {
        "metric": METRIC, "value": value, "unit": "Pauli strings/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": label, "N": n, "batch": b, "alphas": alphas, "seed": seed,
                   "shards": f"{world} state shards" if by_state else f"{world} X-string shards",
                   "l2": "flushed between steps (256 MiB write)",
                   "step": "partial_sums over all 2^N X-strings + allreduce + finalize"},
        "roofline": roof,
        "fwht_hbm_equiv": {"GBps_per_gpu": hbm_equiv, "frac_of_hbm": hbm_equiv / peaks["hbm_gbs"],
                           "note": "16 B/Pauli string workspace write+read, vs measured HBM copy bandwidth"},
        "gpu_launches": int(launches),
        "clocks": clk,
        "e2e": e2e,
        "result": {"M": [float(x) for x in m[0]], "lost_norm": float(ln[0])},
        "profile": prof,
    }
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        line["cpu_baseline"] = cpu_sample(args.config)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
