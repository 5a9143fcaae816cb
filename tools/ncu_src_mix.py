"""Aggregate ncu source-page (SASS) stall samples by opcode: python tools/ncu_src_mix.py src.csv"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
off = 0 if "Source" in rows[0] else 1
h = rows[off]; data = rows[off + 1:]
iS = h.index("Source"); ie = h.index("Instructions Executed")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = collections.defaultdict(lambda: collections.Counter())
cnt = collections.Counter()
for r in data:
    op = r[iS].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    cnt[o] += int(r[ie] or 0)
    for c in cols:
        agg[o][c] += int(r[h.index(c)] or 0)
tot = sum(sum(a.values()) for a in agg.values())
print("opcode  executed  samples%  top stalls")
for o, a in sorted(agg.items(), key=lambda x: -sum(x[1].values()))[:25]:
    s = sum(a.values())
    print(f"{o:10s} {cnt[o]:12d} {100*s/tot:6.1f}%  " + ", ".join(f"{k[6:]} {100*v/tot:.1f}" for k, v in a.most_common(4)))
