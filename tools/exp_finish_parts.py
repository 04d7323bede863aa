"""Finish-stage cost split on M5 (1M x n = 128): staging only (no refine, no schedule), + replay and
schedule output, + refinement.  python tools/exp_finish_parts.py [instances]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_13601_b200 import far, inputs  # noqa: E402

I = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
w = inputs.WORKLOADS["M5"]
tab = torch.from_numpy(inputs.synthetic_parallel(w.profile, w.n, I, w.seed, scaling=w.scaling, times=w.times)).cuda()
F = far.Far(w.profile, w.costs())
ms = torch.empty(I, dtype=torch.int32, device="cuda")
sd = torch.empty((I, w.n, 8), dtype=torch.uint8, device="cuda")
rs = torch.empty((I, 56), dtype=torch.uint8, device="cuda")
cases = [("staging only", dict(flags=far.NO_REFINE | far.NO_SCHEDULE)),
         ("staging+replay, no schedule write (refine 0 it)", dict(max_iterations=0, flags=far.NO_SCHEDULE)),
         ("staging+replay+schedule", dict(max_iterations=0)),
         ("full", dict())]
for name, kw in cases:
    for _ in range(2):
        F.solve_many(tab, out=(ms, sd, rs), **kw)
    torch.cuda.synchronize()
    F.stage_times()
    F.stage_timing(True)
    for _ in range(3):
        F.solve_many(tab, out=(ms, sd, rs), **kw)
    torch.cuda.synchronize()
    F.stage_timing(False)
    n, st = F.stage_times()
    print(name, round(st["finish"] / n, 3), flush=True)
