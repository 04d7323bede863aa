"""Experiment: one far_solve_many over 1M M5 instances vs the same instances split into chunks
solved on two CUDA streams concurrently (kernels of different chunks may co-reside on the SMs)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_13601_b200 import far, inputs  # noqa: E402

w = inputs.WORKLOADS["M5"]
tab = torch.from_numpy(w.table(parallel=True)).cuda()
I = tab.shape[0]
F = far.Far(w.profile, w.costs())
ms = torch.empty(I, dtype=torch.int32, device="cuda")
sd = torch.empty((I, w.n, 8), dtype=torch.uint8, device="cuda")
rs = torch.empty((I, 56), dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]


def run(chunks, nstreams):
    step = -(-I // chunks)
    cur = torch.cuda.current_stream()
    for s in streams[:nstreams]:
        s.wait_stream(cur)
    for c in range(chunks):
        lo, hi = c * step, min(I, (c + 1) * step)
        F.solve_many(tab[lo:hi], stream=streams[c % nstreams], out=(ms[lo:hi], sd[lo:hi], rs[lo:hi]))
    for s in streams[:nstreams]:
        cur.wait_stream(s)


for chunks, ns in ((1, 1), (2, 2), (4, 2), (8, 2), (4, 4)):
    for _ in range(2):
        run(chunks, ns)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run(chunks, ns)
    e1.record()
    torch.cuda.synchronize()
    print(f"chunks {chunks} streams {ns}: {e0.elapsed_time(e1) / 5:.3f} ms per 1M")
