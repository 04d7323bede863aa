"""Per-stage device times of far_solve_many on a workload (C-ABI far_stage_times):
python tools/stage_split.py M3 [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2507_13601_b200 import far, inputs  # noqa: E402

w = inputs.WORKLOADS[sys.argv[1]]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
d = torch.from_numpy(w.table(parallel=True)).cuda()
F = far.Far(w.profile, w.costs())
out = (torch.empty(d.shape[0], dtype=torch.int32, device="cuda"),
       torch.empty((d.shape[0], w.n, 8), dtype=torch.uint8, device="cuda"),
       torch.empty((d.shape[0], 56), dtype=torch.uint8, device="cuda"))
F.solve_many(d, out=out)
torch.cuda.synchronize()
F.stage_times()
F.stage_timing(True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    F.solve_many(d, out=out)
b.record()
torch.cuda.synchronize()
k, st = F.stage_times()
print(w.name, f"{a.elapsed_time(b) / reps:.3f} ms/call", {s: round(v / k, 3) for s, v in st.items() if v > 0})
