"""Regenerate the round's profiles/ files (and profiles/ncu_issue_M5.json) from one GPU session's raw outputs:
  python tools/make_profiles.py ROUND REPORT.ncu-rep LAUNCHES.csv BENCH.json
writes profiles/ncu_traffic_M5.json, profiles/<ROUND>_ncu_final_raw.txt,
profiles/<ROUND>_ncu_source_top_lines.txt, profiles/<ROUND>_launches.csv, profiles/<ROUND>_bench_full.json
and prints the per-kernel table used in profiles/<ROUND>_ncu_summary.md."""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd, rep, launches, bench = sys.argv[1:5]
P = os.path.join(ROOT, "profiles")
py = sys.executable

traffic = subprocess.run([py, os.path.join(ROOT, "tools", "ncu_traffic.py"), rep, "200000", "M5_A100_n128_1M"],
                         capture_output=True, text=True, check=True).stdout
tj = json.loads(traffic)
tj["source"] = (f"ncu --set full capture of one far_solve_many chain, 200k M5 instances "
                f"(profiles/{rnd}_ncu_summary.md)")
json.dump(tj, open(os.path.join(P, "ncu_traffic_M5.json"), "w"), indent=1)
# hardware view for bench.py's roofline.stages_hw: issued lane-ops (warp instructions x active lanes
# per instruction) per instance of each kernel
# (the bench's "prep" stage spans both prep launches: the monotone pass and the general pass)
lane_ops, warp_inst = {}, {}
for k in tj["kernels"]:
    st = "prep" if k["stage"] == "prep_general" else k["stage"]
    lane_ops[st] = lane_ops.get(st, 0.0) + k["warp_inst_per_instance"] * k["thread_inst_per_inst"]
    warp_inst[st] = warp_inst.get(st, 0.0) + k["warp_inst_per_instance"]
issue = {"workload": tj["workload"], "source": tj["source"], "lane_ops_per_instance": lane_ops,
         "warp_inst_per_instance": warp_inst}
json.dump(issue, open(os.path.join(P, "ncu_issue_M5.json"), "w"), indent=1)

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio"]
out = ["# ncu --set full --clock-control none, one far_solve_many chain on 200k M5 instances (A100, n=128, seed 5)",
       "# columns: one per kernel in launch order (prep, prep_general, member0, members, winner, finish, overflow)"]
for k in keys:
    if k in hdr:
        i = hdr.index(k)
        out.append(f"{k:80s} [{units[i]}] " + " | ".join(r[i] for r in rows[2:]))
open(os.path.join(P, f"{rnd}_ncu_final_raw.txt"), "w").write("\n".join(out) + "\n")

top = []
for skip, name in ((0, "far_prep_kernel<5, true> (prep)"), (2, "far_member0_kernel<5> (member0)"),
                   (3, "far_members_kernel<5> (members)"), (5, "far_finish_lane_kernel<5> (finish)")):
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                          "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
    tmp = os.path.join("/tmp", f"src_{skip}.csv")
    open(tmp, "w").write(src)
    lines = subprocess.run([py, os.path.join(ROOT, "tools", "ncu_src.py"), tmp, "25", "--stalls"],
                           capture_output=True, text=True).stdout
    top.append(f"# hottest CUDA source lines, {name}, 200k M5 instances\n{lines}")
open(os.path.join(P, f"{rnd}_ncu_source_top_lines.txt"), "w").write("\n".join(top))
shutil.copy(launches, os.path.join(P, f"{rnd}_launches.csv"))
shutil.copy(bench, os.path.join(P, f"{rnd}_bench_full.json"))

b = json.load(open(bench))
st = b["roofline"]["stages_ms_per_step"]
for k in tj["kernels"]:
    nm = k["name"].replace("void ", "").replace("(KParams)", "").replace("(PParams)", "")
    print(f"| {k['stage']} | `{nm}` | {st.get(k['stage'], 0) if k['stage'] != 'prep_general' else 0:.2f} | {k['ms_cold_serialised']:.3f} | {k['registers']} | "
          f"{k['warps_active_pct']:.0f} % | {k['issue_active_pct']:.0f} % | {k['thread_inst_per_inst']:.1f} | "
          f"{k['dram_read_bytes_per_instance']:.0f} / {k['dram_write_bytes_per_instance']:.0f} |")
print(f"total DRAM per instance: {tj['dram_read_bytes_per_instance']:.0f} + {tj['dram_write_bytes_per_instance']:.0f} B;"
      f" bench {b['value'] / 1e6:.1f} M/s, {b['ms_per_step']:.2f} ms/step")
