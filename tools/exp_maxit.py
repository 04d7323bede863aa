"""Finish-stage time vs the Alg. 2 iteration limit on M5 (1M x n = 128): how much of finish is the
refinement's tail.  python tools/exp_maxit.py [instances]"""
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
for mi in (100, 12, 9, 6, 4, 2, 1, 0):
    for _ in range(2):
        F.solve_many(tab, out=(ms, sd, rs), max_iterations=mi)
    torch.cuda.synchronize()
    F.stage_times()
    F.stage_timing(True)
    for _ in range(3):
        F.solve_many(tab, out=(ms, sd, rs), max_iterations=mi)
    torch.cuda.synchronize()
    F.stage_timing(False)
    n, st = F.stage_times()
    res = far.results_np(rs)
    print(mi, {k: round(v / max(n, 1), 3) for k, v in st.items()}, "mean iters", float(res["iterations"].mean()),
          "evals", float(res["evals"].mean()), flush=True)
