"""Top SASS lines of an ncu source-page CSV (plain or .gz) by a column:
python tools/ncu_src_top.py src.csv[.gz] "<column>" [n]   e.g. "L1 Wavefronts Shared Excessive"."""
import csv, gzip, io, sys
f = sys.argv[1]
txt = (gzip.open(f, "rt") if f.endswith(".gz") else open(f)).read()
rows = list(csv.reader(io.StringIO(txt)))
off = 0 if "Source" in rows[0] else 1
h = rows[off]; data = rows[off + 1:]
col = h.index(sys.argv[2]); n = int(sys.argv[3]) if len(sys.argv) > 3 else 20
iS, iA, iE = h.index("Source"), h.index("Address"), h.index("Instructions Executed")
iW = h.index("Warp Stall Sampling (All Samples)")
val = lambda r: float(r[col] or 0)
tot = sum(val(r) for r in data)
print(f"total {sys.argv[2]}: {tot:.0f}")
for k, r in sorted(enumerate(data), key=lambda x: -val(x[1]))[:n]:
    print(f"{k:5d} {val(r):12.0f} {100 * val(r) / max(tot, 1):5.1f}%  exec {r[iE]:>10s} samp {r[iW]:>6s}  {r[iS].strip()[:70]}")
