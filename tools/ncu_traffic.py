"""Per-kernel DRAM traffic per instance from an ncu --set full capture of one far_solve_many
launch chain: python tools/ncu_traffic.py report.ncu-rep INSTANCES WORKLOAD > profiles/ncu_traffic_<W>.json
Kernels are mapped to the bench's FAR_STAGE_* stages by name (the winner stage is two launches: the
k* != 0 scan and the re-simulations)."""
import csv
import io
import json
import subprocess
import sys

rep, inst, workload = sys.argv[1], int(sys.argv[2]), sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
col = {h: i for i, h in enumerate(hdr)}
STAGE_OF = [("far_prep_kernel<5, 1>", "prep"), ("far_prep_kernel<3, 1>", "prep"), ("far_prep_kernel<", "prep_general"),
            ("far_member0_kernel", "member0"), ("far_members_kernel", "members"), ("far_winner_scan_kernel", "winner"),
            ("far_winner_kernel", "winner"), ("far_finish_lane_kernel", "finish"), ("far_solve_kernel", "overflow")]


def stage_of(name, k):
    for pat, st in STAGE_OF:
        if pat in name:
            return st
    return f"k{k}"


scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
out = {"workload": workload, "source": rep, "instances_per_launch": inst, "kernels": []}
tot_r = tot_w = tot_t = 0.0
for k, r in enumerate(rows[2:]):
    def val(m):
        return float(r[col[m]].replace(",", "")) * scale.get(units[col[m]], 1)
    rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
    t = float(r[col["gpu__time_duration.sum"]]) * {"ms": 1e-3, "us": 1e-6, "ns": 1e-9}[units[col["gpu__time_duration.sum"]]]
    tot_r, tot_w, tot_t = tot_r + rd, tot_w + wr, tot_t + t
    out["kernels"].append({"stage": stage_of(r[col["Kernel Name"]], k), "name": r[col["Kernel Name"]],
                           "grid": r[col["Grid Size"]], "block": r[col["Block Size"]],
                           "registers": int(float(r[col["launch__registers_per_thread"]])),
                           "ms_cold_serialised": t * 1e3,
                           "dram_read_bytes_per_instance": rd / inst, "dram_write_bytes_per_instance": wr / inst,
                           "warps_active_pct": float(r[col["sm__warps_active.avg.pct_of_peak_sustained_active"]]),
                           "issue_active_pct": float(r[col["smsp__issue_active.avg.pct_of_peak_sustained_active"]]),
                           "thread_inst_per_inst": float(r[col["smsp__thread_inst_executed_per_inst_executed.ratio"]]),
                           "warp_inst_per_instance": val("smsp__inst_executed.sum") / inst})
out["dram_read_bytes_per_instance"] = tot_r / inst
out["dram_write_bytes_per_instance"] = tot_w / inst
out["chain_ms_cold_serialised"] = tot_t * 1e3
print(json.dumps(out, indent=1))
