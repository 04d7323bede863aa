"""Time far_solve_many on non-monotone runtime tables (inputs.uniform_random, 100k x A100 x n) against
the monotone generator (A/B helper: FAR_OLD_PREP=1 selects the general prep kernel)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_13601_b200 import far, inputs  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
I = 100_000
F = far.Far("A100")
for name, tab in (("monotone", inputs.synthetic("A100", n, I, 5)), ("uniform", inputs.uniform_random("A100", n, I, 5))):
    d = torch.from_numpy(tab).cuda()
    for _ in range(2):
        F.solve_many(d)
    torch.cuda.synchronize()
    F.stage_timing(True)
    F.stage_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        F.solve_many(d)
    e1.record()
    torch.cuda.synchronize()
    k, st = F.stage_times()
    F.stage_timing(False)
    print(f"{name:9s} n={n}: {e0.elapsed_time(e1) / 3:.3f} ms per 100k;",
          {s: round(v / max(k, 1), 3) for s, v in st.items() if v > 0})
