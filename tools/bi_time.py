import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2507_13601_b200 import far, inputs
w = inputs.WORKLOADS["M5"]
d = torch.from_numpy(w.table(count=100_000, parallel=True)).cuda()
F = far.Far(w.profile, w.costs())
for _ in range(3): F.solve_many(d, flags=far.BEST_IMPROVEMENT)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5): F.solve_many(d, flags=far.BEST_IMPROVEMENT)
b.record(); torch.cuda.synchronize()
print(os.environ.get("FAR_LIB_OVERRIDE", "?")[-10:], round(a.elapsed_time(b) / 5, 3), "ms / 100k")
