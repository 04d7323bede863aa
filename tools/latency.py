import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2507_13601_b200 import far, inputs
for wn in ("M1", "M2", "M3", "M5"):
    w = inputs.WORKLOADS[wn]
    F = far.Far(w.profile, w.costs())
    one = np.ascontiguousarray(w.table(count=1))
    lat = []
    for r in range(220):
        t0 = time.perf_counter(); F.solve_many_host(one)
        if r >= 20: lat.append(time.perf_counter() - t0)
    print(wn, f"{np.median(lat)*1e6:.1f} us")
