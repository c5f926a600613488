"""Per-launch DRAM traffic of the bench's dominant kernel from `ncu --set full` raw CSV exports.

    python tools/ncu_traffic.py out.json CONFIG:KIND:raw.csv[:skip_regex] ...

For each CONFIG (bench.py config name) and KIND (the bench's launch kind: pass_a, pass_b, ...),
averages dram__bytes_read.sum + dram__bytes_write.sum over the captured launches whose kernel
name does NOT match skip_regex (e.g. the final pass of a mixed-mana sweep, which is pass_b).
bench.py reads the JSON and reports it as roofline.traffic next to the algorithmic bytes.
"""
import csv
import io
import json
import re
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    rows = list(csv.reader(io.StringIO(open(path).read())))
    hdr, units = rows[0], dict(zip(rows[0], rows[1]))
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            b += float(d[k].replace(",", "")) * UNIT[units[k]]
        yield d["Kernel Name"], int(d["launch__grid_size"]), b, float(d["gpu__time_duration.sum"].replace(",", ""))


def main():
    out = {}
    for spec in sys.argv[2:]:
        cfg, kind, path, *skip = spec.split(":")
        sel = [(n, g, b, t) for n, g, b, t in launches(path) if not (skip and re.search(skip[0], n))]
        if not sel:
            raise SystemExit(f"{spec}: no launches selected")
        out[cfg] = {"kind": kind, "dram_bytes_per_launch": sum(s[2] for s in sel) / len(sel),
                    "launches": len(sel), "kernels": sorted({s[0][:80] for s in sel}),
                    "grids": sorted({s[1] for s in sel}),
                    "source": f"ncu --set full --clock-control none (cache flushed per launch), {path.split('/')[-1]}"}
    with open(sys.argv[1], "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
