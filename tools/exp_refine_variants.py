"""Oracle-only experiment (CPU): does refining every family member (instead of k* only, R13) or
measuring p_ref against a^1 alone explain the gap to the paper's Table 6?  100 instances per cell."""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from oracle import oracle as O
from paper_2507_13601_b200 import inputs
from fractions import Fraction
O.build()
costs = inputs.reconfig_costs("A100")
for sc, tm in [("poor","narrow"),("mixed","wide"),("good","narrow")]:
  for n in (10, 20, 30):
    tab = inputs.synthetic("A100", n, 100, 6000+n, scaling=sc, times=tm)
    pr_lit = []; pr_all = []; pr_alloc1=[]
    for i in range(tab.shape[0]):
        o = O.far("A100", costs, tab[i])
        ms, ms2 = o["result"]["makespan"], o["result"]["makespan_phase2"]
        pr_lit.append(ms2/ms - 1)
        fam = O.family("A100", tab[i])
        best = None
        for a in fam:
            sa = O.schedule_allocation("A100", costs, tab[i], a)
            r = O.refine("A100", costs, tab[i], sa["slots"], sa["makespan"])
            m = r["result"]["makespan"]
            best = m if best is None else min(best, m)
        pr_all.append(ms2/best - 1)
        # no-ref = first allocation only (a^1) ?
        s1 = O.schedule_allocation("A100", costs, tab[i], fam[0])
        pr_alloc1.append(s1["makespan"]/ms - 1)
    print(sc, tm, n, "p_ref literal %.2f  refine-all-members %.2f  vs a1-only %.2f" % (100*np.mean(pr_lit), 100*np.mean(pr_all), 100*np.mean(pr_alloc1)))
