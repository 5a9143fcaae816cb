"""Write profiles/<round>/<tag>_ncu_summary.txt and the traffic entries bench.py reads from an
`ncu --set full` report (one entry per kernel in the report).

Usage: python profiles/make_summary.py <report.ncu-rep | raw-page .csv> <round dir> <tag> <key prefix>
       e.g.  ... gpurun_out/r2g_large.ncu-rep r2 r2g_large large/tf32x3/staged-{stage}/2
`{stage}` is replaced by covariance / solve / apply / fused (from the kernel name), giving the
keys bench.py uses: "<config>/<precision>/staged-<stage>/<cubes>" or "<config>/<precision>/fused/<cubes>"."""
import csv
import io
import json
import os
import subprocess
import sys

rep, rnd, tag, key = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
HERE = os.path.dirname(os.path.abspath(__file__))
if rep.endswith(".csv"):  # the raw page exported on the GPU box (ncu -i X.ncu-rep --page raw --csv)
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.sum.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg.per_second"]
STAGE = {"chol_kernel": "solve", "solve_small_kernel": "solve", "cov_tc_kernel": "covariance", "cov_kernel": "covariance",
         "apply_tc_kernel": "apply", "apply_kernel": "apply", "fused_kernel": "fused", "doppler": "front_end"}
lines = [f"# ncu --set full --clock-control none --import-source on: {os.path.basename(rep)}"]
entries = {}
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units))
    name = d.get("Kernel Name", "")
    lines.append("== " + name[:140])
    for k in want:
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
    b = sum(float(d[k].replace(",", "")) * scale.get(u[k], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    lines.append(f"  dram read + write per launch: {b:.4g} bytes")
    stage = next((v for k, v in STAGE.items() if k in name), "kernel")
    k = key.replace("staged-{stage}", "fused" if stage == "fused" else f"staged-{stage}").replace("{stage}", stage)
    entries[k] = {"bytes_per_launch": b, "kernel": name[:80], "source": f"profiles/{rnd}/{tag}_ncu_summary.txt"}
os.makedirs(os.path.join(HERE, rnd), exist_ok=True)
open(os.path.join(HERE, rnd, f"{tag}_ncu_summary.txt"), "w").write("\n".join(lines) + "\n")
tj = os.path.join(HERE, "traffic.json")
data = json.load(open(tj)) if os.path.exists(tj) else {}
data.update(entries)
json.dump(data, open(tj, "w"), indent=1)
print("\n".join(lines))
