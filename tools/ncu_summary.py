"""Summarise an .ncu-rep: key throughput metrics and top stall reasons per kernel.
    python tools/ncu_summary.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
if rep.endswith(".csv"):
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed", "smem wavefronts %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2 %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "ld bank conflicts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "st bank conflicts"),
]
for row in rows[2:]:
    d = dict(zip(hdr, row))
    print(f"== {d.get('Kernel Name', '?')[:60]}  (grid {d.get('launch__grid_size')}, block {d.get('launch__block_size')})")
    units = dict(zip(hdr, rows[1]))
    for k, label in keys:
        if k in d:
            print(f"   {label:22s} {d[k]} {units.get(k, '')}")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("   stalls/issue:", ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))
