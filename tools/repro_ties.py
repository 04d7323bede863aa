import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2507_13601_b200 import far, inputs
from oracle import oracle as O
n, count, seed, hi = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
prof = sys.argv[5] if len(sys.argv) > 5 else "H100"
tab = inputs.monotone_ties(prof, n, count, seed, hi=hi)
F = far.Far(prof, inputs.reconfig_costs(prof))
ms, sd, rs = F.solve_many(torch.from_numpy(tab).cuda(), flags=far.GROW_TIES | far.NO_REFINE)
torch.cuda.synchronize()
K = [len(O.family(prof, t, flags=O.GROW_TIES)) for t in tab]
oms, _ = O.far_many(prof, inputs.reconfig_costs(prof), tab, flags=O.GROW_TIES | O.NO_REFINE)
print("n", n, "ok", (ms.cpu().numpy() == oms).all(), "K", K)
