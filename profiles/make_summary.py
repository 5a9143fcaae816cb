"""Write profiles/<tag>_ncu_summary.txt and update profiles/traffic.json from an ncu --set full report.
Usage: python profiles/make_summary.py <report.ncu-rep> <tag> <workload key> [kernel substring for the traffic entry]"""
import csv, io, json, os, subprocess, sys

rep, tag, key = sys.argv[1], sys.argv[2], sys.argv[3]
HERE = os.path.dirname(os.path.abspath(__file__))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__inst_executed.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second"]
lines = [f"# ncu --set full --clock-control none summary: {os.path.basename(rep)}"]
traffic = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    lines.append("== " + d.get("Kernel Name", "")[:120])
    for k in want[1:]:
        if k in d:
            lines.append(f"  {k:70s} {d[k]} {u.get(k, '')}")
    st = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v.replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    st.sort(reverse=True)
    lines.append("  stalls per issue: " + ", ".join(f"{n}={v:.2f}" for v, n in st[:8]))
    b = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        b += float(d[k].replace(",", "")) * scale.get(u[k], 1)
    traffic[d.get("Kernel Name", "")[:60]] = b
open(os.path.join(HERE, f"{tag}_ncu_summary.txt"), "w").write("\n".join(lines) + "\n")
tj = os.path.join(HERE, "traffic.json")
data = json.load(open(tj)) if os.path.exists(tj) else {}
sel = [k for k in traffic if len(sys.argv) > 4 and sys.argv[4] in k] or list(traffic)
kern = max(sel, key=traffic.get)
data[key] = {"bytes_per_launch": traffic[kern], "kernel": kern, "report": tag}
json.dump(data, open(tj, "w"), indent=1)
print("\n".join(lines))
