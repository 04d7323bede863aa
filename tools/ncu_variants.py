"""One launch each of the two variant kernels for an ncu capture (profiles/r1_ncu_variants.md):
the best-improvement warp finish (FAR_BEST_IMPROVEMENT, 100k M5 instances) and the multi-target
forest kernel (A100 x 4, n = 64, 100k batches)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2507_13601_b200 import far, inputs  # noqa: E402

dev = torch.device("cuda:0")
w = inputs.WORKLOADS["M5"]
d = torch.from_numpy(w.table(count=100_000, parallel=True)).to(dev)
F = far.Far(w.profile, w.costs())
r = F.solve_many(d, flags=far.BEST_IMPROVEMENT)[2]
torch.cuda.synchronize()
ev = far.results_np(r)["evals"].sum()
print("best-improvement evals", int(ev))
G = far.Far("A100x4", inputs.reconfig_costs("A100"))
d2 = torch.from_numpy(inputs.synthetic_parallel("A100", 64, 100_000, 6)).to(dev)
G.solve_many(d2)
torch.cuda.synchronize()
print("forest done")
