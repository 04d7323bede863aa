"""Time multi-target FAR (far_forest_kernel) on 100k batches of n = 64 over A100 x 4 and A30 x 2."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_13601_b200 import far, inputs  # noqa: E402

for prof, base in (("A100x4", "A100"), ("A30x2", "A30")):
    tab = torch.from_numpy(inputs.synthetic(base, 64, 100_000, 6)).cuda()
    F = far.Far(prof, inputs.reconfig_costs(base))
    for _ in range(2):
        F.solve_many(tab)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        F.solve_many(tab)
    e1.record()
    torch.cuda.synchronize()
    print(prof, f"{e0.elapsed_time(e1) / 3:.3f} ms per 100k")
