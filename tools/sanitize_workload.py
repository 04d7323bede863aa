"""Small workload that launches every kernel of libfar.so (for compute-sanitizer; tools/sanitize.sh).

Covers, on the A30 and A100 trees: the pipelined chain (far_prep_kernel for n <= 128 and the
PIPE_PREP instantiation for n > 128 / FAR_GROW_TIES, member0, members, winner, the thread finish and,
with FAR_BEST_IMPROVEMENT / n > 256, the warp finish), the fused kernel (small batches,
schedule_batch, local_search, FAR_SWITCH_COST) and its overflow pass (non-monotone inputs), the
multi-target forest kernel, the stream fold, events / validation, lower bounds, the host-memory
pipeline and the peak microbenchmark.  Every flag appears at least once.  Results are checked
against the oracle on a sample (a sanitizer run must also be a correct run)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402
from paper_2507_13601_b200 import far, inputs  # noqa: E402

dev = torch.device("cuda:0")
quick = "--quick" in sys.argv
fl = far
FLAGS = [0, fl.EXHAUSTIVE, fl.NONEMPTY_ALT, fl.GROW_TIES, fl.BEST_IMPROVEMENT, fl.NO_GUARD | fl.NO_REFINE,
         fl.ZERO_RECONFIG, fl.SWITCH_COST, fl.NO_SCHEDULE]
checked = 0


def check(profile, costs, tab, ms, flags, k=4):
    global checked
    oms, _ = O.far_many(profile, costs, tab[:k], flags=flags & ~fl.NO_SCHEDULE)
    assert (ms[:k] == oms).all(), (profile, flags)
    checked += k


for profile in ("A30", "A100"):
    costs = inputs.reconfig_costs(profile)
    F = far.Far(profile, costs)
    for n, I in ((12, 300), (40, 260), (129, 256)) if not quick else ((12, 300),):
        tab = inputs.synthetic(profile, n, I, 7 + n)
        d = torch.from_numpy(tab).to(dev)
        for flags in FLAGS if not quick else (0, fl.BEST_IMPROVEMENT):
            ms, _, _ = F.solve_many(d, flags=flags)
            torch.cuda.synchronize()
            check(profile, costs, tab, ms.cpu().numpy(), flags)
        # fused kernel (small batch), overflow pass (non-monotone), host pipeline
        ms, _, _ = F.solve_many(d[:40])
        u = inputs.uniform_random(profile, n, 300, 3)
        ms2, _, _ = F.solve_many(torch.from_numpy(u).to(dev))
        torch.cuda.synchronize()
        check(profile, costs, tab, ms.cpu().numpy(), 0)
        check(profile, costs, u, ms2.cpu().numpy(), 0)
        msh, _, _ = F.solve_many_host(np.ascontiguousarray(tab))
        check(profile, costs, tab, msh, 0)
    # single batch + local search (fused, MODE_LOCAL)
    t1 = inputs.synthetic(profile, 20, 1, 5)[0]
    slots, r = F.schedule_batch(t1)
    s2, r2 = F.local_search(t1, slots, makespan_phase2=int(r["makespan"]))
    # n > 256: warp finish
    if not quick:
        tb = inputs.synthetic(profile, 300, 8, 9)
        ms, _, _ = F.solve_many(torch.from_numpy(tb).to(dev))
        torch.cuda.synchronize()
        check(profile, costs, tb, ms.cpu().numpy(), 0, k=2)
    # streams (fused solve of every batch + the fold), events + validation, lower bounds
    st = inputs.synthetic(profile, 16, 3 * 4, 11).reshape(3, 4, 16, -1)
    F.concat_streams(torch.from_numpy(np.ascontiguousarray(st)).to(dev))
    F.concat_streams(torch.from_numpy(np.ascontiguousarray(st)).to(dev), flags=fl.NO_SEAM_MOVES)
    d = torch.from_numpy(inputs.synthetic(profile, 24, 64, 13)).to(dev)
    ms, sd, _ = F.solve_many(d)
    ev, nev, _ = F.schedule_events(d, sd)
    viol = F.validate_schedules(d, sd, ev, nev)
    F.lower_bounds(d)
    torch.cuda.synchronize()
    assert int(viol.sum()) == 0
    F.sync()
    F.close()
    # multi-target forest
    G = far.Far(profile + "x2", costs)
    tg = inputs.synthetic(profile, 20, 40, 17)
    dg = torch.from_numpy(tg).to(dev)
    _, sg, _ = G.solve_many(dg)
    G.solve_many(dg, flags=fl.BEST_IMPROVEMENT)
    # events + validator on the forest (far_forest_check.cuh)
    evg, nevg, _ = G.schedule_events(dg, sg)
    violg = G.validate_schedules(dg, sg, evg, nevg)
    torch.cuda.synchronize()
    assert int(violg.sum()) == 0
    G.sync()
    G.close()

P = far.Far("A100")
for mode in (0, 1, 2):
    P.measure_peak(mode)
P.close()
print(f"sanitize workload OK ({checked} instances checked against the oracle)")
