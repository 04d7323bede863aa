"""Stage split of far_concat_streams on ONE M4 stream (64 batches x 64 tasks) per tree: the
latency view of config 4."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_13601_b200 import far, inputs  # noqa: E402

for prof in ("A30", "A100"):
    S, B, n = 1, 64, 64
    tab = inputs.synthetic(prof, n, S * B, 4).reshape(S, B, n, -1)
    d = torch.from_numpy(np.ascontiguousarray(tab)).cuda()
    F = far.Far(prof)
    for _ in range(3):
        F.concat_streams(d)
    torch.cuda.synchronize()
    F.stage_timing(True)
    F.stage_times()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        F.concat_streams(d)
    e1.record()
    torch.cuda.synchronize()
    k, st = F.stage_times()
    print(prof, f"{e0.elapsed_time(e1) / 5:.3f} ms", {s: round(v / max(k, 1), 3) for s, v in st.items() if v > 0}, k)
    for flags in (far.NO_SEAM_MOVES,):
        for _ in range(2):
            F.concat_streams(d, flags=flags)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            F.concat_streams(d, flags=flags)
        e1.record()
        torch.cuda.synchronize()
        print(prof, "no seam moves", f"{e0.elapsed_time(e1) / 5:.3f} ms")
