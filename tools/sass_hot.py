"""Group SASS lines of an ncu source page by region: print instruction-mix and stall samples (dev helper)."""
import csv, sys, re, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) >= len(hdr) - 2 and r[0].startswith("0x")]
tot_exec = sum(int(r[idx["Instructions Executed"]] or 0) for r in data)
tot_samp = sum(int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
print("total warp-instr executed", tot_exec, "samples", tot_samp)
mix = collections.Counter(); samp = collections.Counter()
for r in data:
    op = r[idx["Source"]].strip().split()
    if not op: continue
    o = op[0]
    if o.startswith("@"): o = op[1]
    o = o.split(".")[0]
    mix[o] += int(r[idx["Instructions Executed"]] or 0)
    samp[o] += int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
for o, c in mix.most_common(25):
    print(f"  {o:10s} exec {c/tot_exec*100:6.2f}%  stall-samples {samp[o]/max(tot_samp,1)*100:6.2f}%")
# hottest contiguous regions by samples (window 40 lines)
w = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if w:
    s = [int(r[idx["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
    e = [int(r[idx["Instructions Executed"]] or 0) for r in data]
    blocks = []
    for i in range(0, len(data), w):
        blocks.append((sum(s[i:i+w]), sum(e[i:i+w]), i))
    blocks.sort(reverse=True)
    for sm, ex, i in blocks[:8]:
        print(f"lines {i}-{i+w}: samples {sm/tot_samp*100:5.1f}%  exec {ex/tot_exec*100:5.1f}%   first: {data[i][idx['Source']].strip()[:60]}")
