"""Pins of the oracle's evaluation statistics (oracle.table_stats; PAPER.md P:1057-1066 rho,
P:1209-1212 p_ref) against closed forms and invariants -- not against a retyping of the formula."""
from fractions import Fraction

import numpy as np

from paper_2507_13601_b200 import inputs


def test_rho_is_one_on_perfectly_balanced_instances(O):
    # seven identical perfectly-scaling tasks, zero reconfiguration: a^1 = size 1 (work ties ->
    # smallest size), one task per slice, omega = 700 = baseline (7 * 700 / 7)
    zero = inputs.reconfig_costs("A100", zero=True)
    task = [700, 350, 700 // 3 + 1, 175, 100]
    tab = np.array([[task] * 7], dtype=np.int32)
    st = O.table_stats("A100", zero, tab)
    assert st["rho"] == 1 and st["p_ref"] == 0
    # one perfectly-scaling task: the family reaches size 7, omega = 100 = 700 / 7
    one = np.array([[[700, 350, 234, 175, 100]]], dtype=np.int32)
    assert O.table_stats("A100", zero, one)["rho"] == 1


def test_rho_closed_form_single_task_with_reconfiguration(O):
    # one task with Table 2 costs: omega = min over the family of t_create(s) + t(s).  Works are
    # 7000, 7000, 7002, 7000, 7000: a^1 = 1 (ties -> smallest), then argmin over larger sizes with
    # ties -> smallest: 2, then 4 (7002 > 7000 skips size 3), then 7
    costs = inputs.reconfig_costs("A100")
    t = [7000, 3500, 2334, 1750, 1000]
    cr = [int(x) for x in costs[0]]
    omega = min(cr[c] + t[c] for c in (0, 1, 3, 4))
    st = O.table_stats("A100", costs, np.array([[t]], dtype=np.int32))
    assert st["rho"] == Fraction(omega * 7, 7000)


def test_statistics_bounds_and_mean(O):
    costs = inputs.reconfig_costs("A100")
    tab = inputs.synthetic("A100", 12, 40, 77)
    st = O.table_stats("A100", costs, tab)
    per = [O.table_stats("A100", costs, tab[i:i + 1]) for i in range(tab.shape[0])]
    assert all(p["rho"] >= 1 for p in per)          # baseline is a lower bound
    assert all(p["p_ref"] >= 0 for p in per)        # refinement never worse with the guard
    assert st["rho"] == sum(p["rho"] for p in per) / len(per)
    assert st["p_ref"] == sum(p["p_ref"] for p in per) / len(per)
    # zero-reconfiguration A100 factor 2: rho <= omega_FAR / omega* * omega* / baseline
    zero = inputs.reconfig_costs("A100", zero=True)
    small = inputs.synthetic("A100", 5, 20, 78)
    for i in range(small.shape[0]):
        r = O.table_stats("A100", zero, small[i:i + 1])["rho"]
        w, _ = O.lower_bound("A100", small[i])
        opt = O.bruteforce("A100", small[i])
        assert Fraction(opt * 7, w) <= r <= 2 * Fraction(opt * 7, w)


def test_concat_statistics_closed_forms(O):
    # two perfectly balanced batches (seven identical size-1 tasks each, zero reconfiguration):
    # every slice is busy until T in both, so no reversal or seam move can overlap them and every
    # concatenation gives 2T: p_rev = p_move/swap = 0
    zero = inputs.reconfig_costs("A100", zero=True)
    task = [700, 350, 700 // 3 + 1, 175, 100]
    two = np.array([[[task] * 7, [task] * 7]], dtype=np.int32)
    st = O.concat_stats("A100", zero, two)
    assert st["p_rev"] == 0 and st["p_move_swap"] == 0 and st["moves"] == 0 and st["swaps"] == 0
    assert O.multi_batch_p("A100", zero, two[0]) == 0  # omega = 1400 = baseline (2 * 7 * 700 / 7)
    # a one-batch stream: p_multi = (rho - 1) * 100 of that batch (Tables 4 and 9 share the baseline)
    costs = inputs.reconfig_costs("A100")
    one = inputs.synthetic("A100", 15, 1, 92)
    assert O.multi_batch_p("A100", costs, one) == (O.table_stats("A100", costs, one)["rho"] - 1) * 100
