"""e2e (far_solve_many_host) time on M5 for several host-pipeline chunk sizes: python tools/e2e_sweep.py 48 96 192"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2507_13601_b200 import far, inputs  # noqa: E402

w = inputs.WORKLOADS["M5"]
tab = w.table(parallel=True)
I = tab.shape[0]
hin = torch.from_numpy(tab).pin_memory().numpy()
hms = torch.empty(I, dtype=torch.int32).pin_memory().numpy()
hsd = torch.empty((I, w.n, 8), dtype=torch.uint8).pin_memory().numpy().view(far.SLOT_DT)[..., 0]
hrs = torch.empty((I, 56), dtype=torch.uint8).pin_memory().numpy().view(far.RESULT_DT)[..., 0]
for mb in sys.argv[1:]:
    os.environ["FAR_HOST_CHUNK_MB"] = mb
    F = far.Far(w.profile, w.costs())
    F.solve_many_host(hin, out=(hms, hsd, hrs))
    t0 = time.perf_counter()
    for _ in range(3):
        F.solve_many_host(hin, out=(hms, hsd, hrs))
    dt = (time.perf_counter() - t0) / 3
    print(f"chunk {mb} MB: {dt * 1000:.1f} ms -> {I / dt / 1e6:.2f} M instances/s", flush=True)
    F.close()
