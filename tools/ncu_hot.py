"""Top stall locations from an `ncu --page source --csv --print-source sass` export (gz or plain):
    python tools/ncu_hot.py src.csv.gz [top]
Prints the SASS lines with the most warp-stall samples and the dominant stall reasons of each."""
import csv
import gzip
import io
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
lines = raw.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = 0
recs = []
for r in rows[1:]:
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    tot += s
    st = sorted(((int(r[ix[c]] or 0), c[6:]) for c in stall_cols), reverse=True)[:3]
    recs.append((s, r[ix["Source"]].strip(), st))
by_reason = {}
for r in rows[1:]:
    for c in stall_cols:
        try:
            by_reason[c[6:]] = by_reason.get(c[6:], 0) + int(r[ix[c]] or 0)
        except (ValueError, IndexError):
            pass
print(f"total samples {tot}; by reason:", ", ".join(f"{k}={v / max(tot, 1):.2f}" for k, v in
                                                  sorted(by_reason.items(), key=lambda x: -x[1])[:10]))
for s, src, st in sorted(recs, key=lambda x: -x[0])[:top]:
    print(f"{s / max(tot, 1):6.3f}  {src[:70]:70s} " + " ".join(f"{n}={v}" for v, n in st if v))
