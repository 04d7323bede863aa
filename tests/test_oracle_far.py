"""Oracle pins for phases 1-3: worked examples, the paper's bounds, brute force,
feasibility (constraints 1-3) and invariants.  None of these re-types the
oracle's own formulas; each checks something PAPER.md (or mathematics) fixes."""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

from paper_2507_13601_b200 import inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_traces.json")))
SLICES = {"A30": 4, "A100": 7, "H100": 7}


def _t(x, profile):
    return np.array(x, dtype=np.int32).reshape(-1, len(inputs.SIZES[profile]))


# ----------------------------------------------------------------- worked examples
@pytest.mark.parametrize("case", GOLD["schedule_allocation"], ids=lambda c: c["cite"][:24])
def test_alg1_traces(O, case):
    r = O.schedule_allocation(case["profile"], case["costs"], _t(case["times"], case["profile"]), case["alloc"])
    assert r["makespan"] == case["makespan"]
    assert r["slots"]["start"].tolist() == case["starts"]
    if "events" in case:
        assert [list(map(int, e)) for e in r["events"]] == case["events"]


@pytest.mark.parametrize("case", GOLD["family"], ids=lambda c: c["cite"][:12])
def test_family_examples(O, case):
    fam = O.family(case["profile"], _t(case["times"], case["profile"]))
    assert fam.tolist() == case["family"]


def test_far_example(O):
    case = GOLD["far"][0]
    t = _t(case["times"], case["profile"])
    fam = O.family(case["profile"], t)
    ms = [O.schedule_allocation(case["profile"], None, t, a)["makespan"] for a in fam]
    assert ms == case["member_makespans"]
    r = O.far(case["profile"], None, t)["result"]
    assert r["makespan"] == case["makespan"] and r["alloc_index"] == case["alloc_index"]
    assert O.bruteforce(case["profile"], t) == case["optimum"]


@pytest.mark.parametrize("case", GOLD["refine"], ids=["move", "swap"])
def test_refine_examples(O, case):
    t = _t(case["times"], case["profile"])
    p2 = O.schedule_allocation(case["profile"], None, t, case["alloc"])
    assert p2["makespan"] == case["phase2_makespan"]
    r = O.refine(case["profile"], None, t, p2["slots"], p2["makespan"])
    res = r["result"]
    assert (res["makespan"], res["moves"], res["swaps"]) == (case["makespan"], case["moves"], case["swaps"])
    # the headline evals/s rests on this counter (R27); hand-traced in the golden file (trace_alg2)
    assert (res["evals"], res["iterations"]) == (case["evals"], case["iterations"])
    assert r["slots"]["node"].tolist() == case["nodes"]
    # Fig. 6: > 1.5x ; Fig. 7: almost 1.25x
    ratio = Fraction(case["phase2_makespan"], case["makespan"])
    assert ratio >= Fraction(3, 2) if case["moves"] else Fraction(6, 5) <= ratio < Fraction(5, 4)
    assert O.validate(case["profile"], None, t, r["slots"], r["events"]) == 0


def test_empty_and_single(O):
    for profile in ("A30", "A100"):
        nc = len(inputs.SIZES[profile])
        r = O.far(profile, inputs.reconfig_costs(profile), np.zeros((0, nc), np.int32))
        assert r["result"]["makespan"] == 0 and r["result"]["family_size"] == 0
        # single task, zero reconfiguration, property 1: FAR = t(max size) = min_s t(s)
        for t in inputs.synthetic(profile, 1, 50, 11):
            r = O.far(profile, None, t)["result"]
            assert r["makespan"] == t.min() == t[0, -1]


# ----------------------------------------------------------------- phase 1 invariants
@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_family_invariants(O, profile):
    sizes = inputs.SIZES[profile]
    tabs = [inputs.synthetic(profile, 12, 40, 1), inputs.uniform_random(profile, 12, 40, 2),
            inputs.small_ties(profile, 12, 40, 3), inputs.monotone_ties(profile, 12, 40, 4)]
    for tab in tabs:
        for t in tab:
            fam = O.family(profile, t)
            n = t.shape[0]
            assert 1 <= len(fam) <= 1 + n * (len(sizes) - 1)
            col = {s: j for j, s in enumerate(sizes)}
            a1 = fam[0]
            for i in range(n):  # P:341 argmin work, smallest s on ties
                w = [s * int(t[i, col[s]]) for s in sizes]
                assert a1[i] == sizes[int(np.argmin(w))]
            for k in range(len(fam) - 1):
                d = np.nonzero(fam[k + 1] != fam[k])[0]
                assert len(d) == 1
                j = d[0]
                cur = np.array([t[i, col[fam[k][i]]] for i in range(n)])
                assert cur[j] == cur.max() and j == int(np.argmax(cur))
                assert fam[k + 1][j] > fam[k][j]
            last = fam[-1]
            cur = np.array([t[i, col[last[i]]] for i in range(n)])
            assert last[int(np.argmax(cur))] == sizes[-1]


def test_work_monotone_gives_all_ones(O):
    # if s*t(s) is non-decreasing for every task, a^1 = 1 slice everywhere
    t = np.array([[10, 6, 4], [7, 5, 2], [3, 3, 3]], np.int32)
    assert O.family("A30", t)[0].tolist() == [1, 1, 1]


# ----------------------------------------------------------------- §5 bounds (zero reconfiguration)
def _w_h(t, alloc, sizes):
    col = {s: j for j, s in enumerate(sizes)}
    W = sum(int(a) * int(t[i, col[int(a)]]) for i, a in enumerate(alloc))
    H = max(int(t[i, col[int(a)]]) for i, a in enumerate(alloc))
    return W, H


@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_per_allocation_bounds(O, profile):
    """P:847 (A30): w <= W/4 + 3h/4.  P:898 (A100): w <= max(W/6+5h/6, W/4, W/5+3h/5).
    Checked on every family member and on random allocations, exact integer arithmetic."""
    sizes = inputs.SIZES[profile]
    rng = np.random.default_rng(5)
    tabs = [inputs.synthetic(profile, n, 60, 20 + n) for n in (3, 8, 17)] + \
           [inputs.uniform_random(profile, n, 60, 30 + n) for n in (4, 9)]
    checked = 0
    for tab in tabs:
        for t in tab:
            allocs = list(O.family(profile, t)) + [rng.choice(sizes, t.shape[0]) for _ in range(3)]
            for a in allocs:
                w = O.schedule_allocation(profile, None, t, a)["makespan"]
                W, H = _w_h(t, a, sizes)
                if profile == "A30":
                    assert 4 * w <= W + 3 * H
                else:
                    assert 60 * w <= max(10 * W + 50 * H, 15 * W, 12 * W + 36 * H)
                checked += 1
    assert checked > 1000


@pytest.mark.parametrize("profile,factor", [("A30", Fraction(7, 4)), ("A100", Fraction(2))])
def test_approximation_factor_vs_bruteforce(O, profile, factor):
    """Theorem 1 + §5: with zero reconfiguration and property 1,
    w_FAR <= 7/4 w* (A30), <= 2 w* (A100).  Also LB <= w* <= w_FAR."""
    ns = (2, 3, 4, 5, 6) if profile == "A30" else (2, 3, 4, 5)
    for n in ns:
        for t in inputs.synthetic(profile, n, 40, 100 + n):
            w_far = O.far(profile, None, t)["result"]["makespan"]
            w_opt = O.bruteforce(profile, t)
            W, H = O.lower_bound(profile, t)
            assert W <= SLICES[profile] * w_opt and H <= w_opt <= w_far
            assert w_far <= factor * w_opt


def test_bruteforce_closed_forms(O):
    # identical 1-slice-only tasks (flat times): w* = ceil(n / slices) * t
    for profile in ("A30", "A100"):
        nc = len(inputs.SIZES[profile])
        for n in range(1, 6):
            t = np.full((n, nc), 9, np.int32)
            assert O.bruteforce(profile, t) == -(-n // SLICES[profile]) * 9
    # one task: min over sizes
    t = np.array([[8, 5, 7]], np.int32)
    assert O.bruteforce("A30", t) == 5


# ----------------------------------------------------------------- feasibility and guards
@pytest.mark.parametrize("profile", ["A30", "A100", "H100"])
def test_far_feasible_and_bounded(O, profile):
    costs = inputs.reconfig_costs(profile)
    tabs = [inputs.synthetic(profile, n, 25, 40 + n) for n in (1, 5, 10, 23)] + \
           [inputs.uniform_random(profile, 11, 25, 9), inputs.small_ties(profile, 9, 25, 8)]
    if profile != "A30":
        tabs.append(inputs.rodinia_like(25, 1))
    for tab in tabs:
        for t in tab:
            r = O.far(profile, costs, t)
            res = r["result"]
            assert O.validate(profile, costs, t, r["slots"], r["events"]) == 0
            assert res["makespan"] <= res["makespan_phase2"]          # guard: refinement never worse
            W, H = O.lower_bound(profile, t)
            assert SLICES[profile] * res["makespan"] >= W and res["makespan"] >= H
            nr = O.far(profile, costs, t, flags=O.NO_REFINE)
            assert O.validate(profile, costs, t, nr["slots"], nr["events"]) == 0
            assert nr["result"]["makespan"] == res["makespan_phase2"]
            z = O.far(profile, costs, t, max_iterations=0)
            assert (z["slots"] == nr["slots"]).all() and z["result"]["makespan"] == res["makespan_phase2"]
            assert r["slots"]["start"].tolist() == O.far(profile, costs, t)["slots"]["start"].tolist()


def test_refine_fixpoint_and_balanced(O):
    # replay of the phase-2 tree reproduces phase 2 exactly (O7 fixpoint): refine with 0 iterations
    for t in inputs.synthetic("A100", 14, 30, 77):
        costs = inputs.reconfig_costs("A100")
        p2 = O.far("A100", costs, t, flags=O.NO_REFINE)
        r = O.refine("A100", costs, t, p2["slots"], p2["result"]["makespan"], max_iterations=0)
        assert (r["slots"] == p2["slots"]).all()
    # balanced schedule (all slice ends equal) -> 0 moves, 0 swaps
    t = np.full((4, 3), 5, np.int32)
    r = O.far("A30", None, t)["result"]
    assert r["makespan"] == 5 and r["moves"] == 0 and r["swaps"] == 0


def test_validator_rejects(O):
    """Negative pins for the validator."""
    t = np.array([[2, 2, 2], [2, 2, 2]], np.int32)
    slot = np.zeros(2, O.SLOT_DT)
    ev_dt = [("kind", "<i4"), ("node", "<i4"), ("start", "<i8"), ("dur", "<i8")]
    # two tasks on S0 at [0,2) and [1,3) -> constraint 1
    slot["node"] = [3, 3]; slot["size_used"] = [1, 1]; slot["start"] = [0, 1]
    ev = np.array([(0, 3, 0, 0)], ev_dt)
    assert O.validate("A30", None, t, slot, ev) > 0
    # node 1 ({S0,S1}) and leaf 4 (S1) concurrently -> constraints 1/2
    slot["node"] = [1, 4]; slot["size_used"] = [2, 1]; slot["start"] = [0, 1]
    ev = np.array([(0, 1, 0, 0), (0, 4, 0, 0)], ev_dt)
    assert O.validate("A30", None, t, slot, ev) > 0
    # missing destroy of node 1 before leaf 3 is created -> constraint 3 / lifecycle
    costs = np.array([[1, 1, 1], [1, 1, 1]], np.int32)
    slot["node"] = [1, 3]; slot["size_used"] = [2, 1]; slot["start"] = [1, 5]
    ev = np.array([(0, 1, 0, 1), (0, 3, 3, 1)], ev_dt)
    assert O.validate("A30", costs, t, slot, ev) > 0
    ev = np.array([(0, 1, 0, 1), (1, 1, 3, 1), (0, 3, 4, 1)], ev_dt)
    assert O.validate("A30", costs, t, slot, ev) == 0
    # overlapping reconfiguration events -> constraint 3
    ev = np.array([(0, 1, 0, 1), (1, 1, 3, 1), (0, 3, 3, 1)], ev_dt)
    assert O.validate("A30", costs, t, slot, ev) > 0


def test_input_errors(O):
    with pytest.raises(O.OracleError):
        O.far("A30", None, np.array([[1, 0, 1]], np.int32))        # t < 1
    with pytest.raises(O.OracleError):
        O.far("A30", None, np.full((1025, 3), 1, np.int32))        # n > 1024
    with pytest.raises(O.OracleError):
        O.far(7, None, np.ones((1, 3), np.int32))                  # unknown profile


def test_grow_ties_variant_family(O):
    # two identical perfectly-scaling A30 tasks (work 4 at every size): the literal reading (R2)
    # grows one tied task per step (lowest index), the P:349 formula (FAR_GROW_TIES) grows both
    t = np.array([[4, 2, 1], [4, 2, 1]], dtype=np.int32)
    assert O.family("A30", t).tolist() == [[1, 1], [2, 1], [2, 2], [4, 2], [4, 4]]
    assert O.family("A30", t, flags=O.GROW_TIES).tolist() == [[1, 1], [2, 2], [4, 4]]
    # a tie, then a single longest task that ends the family at the largest size (hand-traced):
    # works of task 2 are 3, 6, 12 -> a^1 = 1; it grows 1 -> 2 -> 4 with t = 3 throughout
    u = np.array([[4, 2, 1], [4, 2, 1], [3, 3, 3]], dtype=np.int32)
    assert O.family("A30", u, flags=O.GROW_TIES).tolist() == [[1, 1, 1], [2, 2, 1], [2, 2, 2], [2, 2, 4]]
    assert O.family("A30", u).tolist() == [[1, 1, 1], [2, 1, 1], [2, 2, 1], [2, 2, 2], [2, 2, 4]]


# ----------------------------------------------------------------- best-improvement variant (R30)
@pytest.mark.parametrize("case", GOLD["refine_best"], ids=lambda c: c["example"])
def test_best_improvement_examples(O, case):
    """Hand traces of the north star's literal phase 3 (R30) on the two Alg. 2 examples."""
    base = next(c for c in GOLD["refine"] if case["example"] in c["cite"])
    t = _t(base["times"], base["profile"])
    p2 = O.schedule_allocation(base["profile"], None, t, base["alloc"])
    r = O.refine(base["profile"], None, t, p2["slots"], p2["makespan"], flags=O.BEST_IMPROVEMENT)
    res = r["result"]
    got = (res["makespan"], res["moves"], res["swaps"], res["evals"], res["iterations"])
    assert got == (case["makespan"], case["moves"], case["swaps"], case["evals"], case["iterations"])
    assert r["slots"]["node"].tolist() == case["nodes"]
    assert O.validate(base["profile"], None, t, r["slots"], r["events"]) == 0


def _laminar_key(lo, hi, S, load):
    """(makespan, #slices reaching it) of a zero-reconfiguration node assignment by the laminar
    closed form (slice end = sum of the loads of the nodes covering the slice),
    computed from scratch -- independent of the oracle's incremental +-t slice ends."""
    e = [sum(load[v] for v in range(len(lo)) if lo[v] <= s < hi[v]) for s in range(S)]
    w = max(e)
    return w, e.count(w)


@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_best_improvement_local_optimum(O, profile):
    """With zero reconfiguration the variant ends in a local optimum of its neighbourhood: no
    same-size move and no swap lowers (makespan, #critical slices), and the replayed makespan is
    the closed-form one."""
    lo, hi, _ = O.nodes(profile)
    lo, hi = lo.tolist(), hi.tolist()
    S = SLICES[profile]
    tabs = [inputs.synthetic(profile, n, 6, 90 + n) for n in (3, 9, 17)] + [inputs.small_ties(profile, 8, 6, 5)]
    for tab in tabs:
        for t in tab:
            r = O.far(profile, None, t, max_iterations=10000, flags=O.BEST_IMPROVEMENT)
            res, sl = r["result"], r["slots"]
            assert res["reverted"] == 0 and res["iterations"] < 10000
            node = sl["node"].tolist()
            dur = [int(t[j][inputs.SIZES[profile].index(int(sl["size_used"][j]))]) for j in range(len(t))]

            def key(nd):
                load = [0] * len(lo)
                for j, v in enumerate(nd):
                    load[v] += dur[j]
                return _laminar_key(lo, hi, S, load)

            cur = key(node)
            assert cur[0] == res["makespan"]
            size = [hi[v] - lo[v] for v in range(len(lo))]
            for j in range(len(t)):
                for u in range(len(lo)):
                    if u != node[j] and size[u] == size[node[j]]:
                        nd = list(node); nd[j] = u
                        assert key(nd) >= cur
                for k in range(j + 1, len(t)):
                    if node[k] != node[j] and size[node[k]] == size[node[j]]:
                        nd = list(node); nd[j], nd[k] = node[k], node[j]
                        assert key(nd) >= cur


@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_best_improvement_feasible_and_guarded(O, profile):
    costs = inputs.reconfig_costs(profile)
    for t in list(inputs.synthetic(profile, 14, 12, 31)) + list(inputs.uniform_random(profile, 10, 8, 3)):
        r = O.far(profile, costs, t, flags=O.BEST_IMPROVEMENT)
        res = r["result"]
        assert O.validate(profile, costs, t, r["slots"], r["events"]) == 0
        assert res["makespan"] <= res["makespan_phase2"]
        z = O.far(profile, costs, t, max_iterations=0, flags=O.BEST_IMPROVEMENT)
        assert z["result"]["makespan"] == res["makespan_phase2"] and z["result"]["evals"] == 0


# ----------------------------------------------------------------- multi-target FAR (NEXT-2, R31)
def test_multi_gpu_forest_model(O):
    """as many trees as GPUs; node ids t*NN + v, slices t*S + [lo, hi)."""
    for base, S, NN in (("A30", 4, 7), ("A100", 7, 13)):
        lo1, hi1, par1 = O.nodes(base)
        for g in (2, 3, 8):
            lo, hi, par = O.nodes(f"{base}x{g}")
            assert len(lo) == g * NN and (par < 0).sum() == g
            for t in range(g):
                assert (lo[t * NN:(t + 1) * NN] == lo1 + t * S).all() and (hi[t * NN:(t + 1) * NN] == hi1 + t * S).all()
    with pytest.raises(O.OracleError):
        O.far("A30x9", None, np.ones((2, 3), np.int32))


def test_multi_gpu_hand_trace(O):
    """Hand trace (A30 x 2, zero reconfiguration): two perfectly scaling tasks t = (4, 2, 1).
    Family [1,1] [2,1] [2,2] [4,2] [4,4]; Alg. 1 with both roots at time 0 gives 4, 4, 2, 2, 1
    (member [4,4] runs each task on its own GPU's root); one A30 gives 4, 4, 2, 3, 2."""
    t = np.array([[4, 2, 1], [4, 2, 1]], np.int32)
    fam = O.family("A30x2", t)
    assert fam.tolist() == [[1, 1], [2, 1], [2, 2], [4, 2], [4, 4]]
    assert [O.schedule_allocation("A30x2", None, t, a)["makespan"] for a in fam] == [4, 4, 2, 2, 1]
    assert [O.schedule_allocation("A30", None, t, a)["makespan"] for a in fam] == [4, 4, 2, 3, 2]
    r = O.far("A30x2", None, t)
    assert r["result"]["makespan"] == 1 and r["result"]["alloc_index"] == 4
    assert r["slots"]["node"].tolist() == [0, 7]


@pytest.mark.parametrize("g", [2, 3])
def test_multi_gpu_a30_bounds(O, g):
    """with g A30s the A30 argument gives, per allocation, 4g*w <= W + (4g-1)*h (zero
    reconfiguration), hence w_FAR <= (8g-1)/(4g) * w*; and LB <= w* <= w_FAR."""
    prof = f"A30x{g}"
    for t in list(inputs.synthetic("A30", 12, 40, 300 + g)) + list(inputs.small_ties("A30", 9, 30, 7)):
        for a in O.family(prof, t):
            ms = O.schedule_allocation(prof, None, t, a)["makespan"]
            W = sum(int(s) * int(t[i][inputs.SIZES["A30"].index(int(s))]) for i, s in enumerate(a))
            h = max(int(t[i][inputs.SIZES["A30"].index(int(s))]) for i, s in enumerate(a))
            assert 4 * g * ms <= W + (4 * g - 1) * h
    for t in inputs.synthetic("A30", 5, 12, 310 + g):
        opt = O.bruteforce(prof, t)
        w = O.far(prof, None, t)["result"]["makespan"]
        Wm, H = O.lower_bound(prof, t)
        assert opt <= w and 4 * g * w <= (8 * g - 1) * opt
        assert 4 * g * opt >= Wm and opt >= H


@pytest.mark.parametrize("prof", ["A30x2", "A100x2", "A100x3", "H100x4"])
def test_multi_gpu_feasible_and_bounded(O, prof):
    base, g = prof.split("x")
    g = int(g)
    costs = inputs.reconfig_costs(base)
    for t in list(inputs.synthetic(base, 20, 12, 320 + g)) + list(inputs.uniform_random(base, 9, 8, 5)):
        for flags in (0, O.BEST_IMPROVEMENT):
            r = O.far(prof, costs, t, flags=flags)
            res = r["result"]
            assert O.validate(prof, costs, t, r["slots"], r["events"]) == 0
            assert res["makespan"] <= res["makespan_phase2"]
            W, H = O.lower_bound(prof, t)
            assert g * SLICES[base] * res["makespan"] >= W and res["makespan"] >= H
    # n <= g identical property-1 tasks, zero reconfiguration: each gets a whole GPU (the last
    # family member), so w_FAR = t(largest size) = the lower bound max_i min_s t_i(s)
    t = np.tile(inputs.synthetic(base, 1, 1, 9)[0], (g, 1))
    assert O.far(prof, None, t)["result"]["makespan"] == int(t[0].min())


# ----------------------------------------------------------------- 4->3 switch-cost variant (R7)
@pytest.mark.parametrize("case", GOLD["switch_cost"], ids=["switch", "create3"])
def test_switch_cost_traces(O, case):
    t = _t(case["times"], case["profile"])
    costs = inputs.reconfig_costs(case["profile"])
    for key, flags in (("default", 0), ("switch", O.SWITCH_COST)):
        r = O.schedule_allocation(case["profile"], costs, t, case["alloc"], flags=flags)
        assert r["makespan"] == case[key]["makespan"], key
        assert r["slots"]["start"].tolist() == case[key]["starts"], key
        assert [list(map(int, e)) for e in r["events"]] == case[key]["events"], key
        assert O.validate(case["profile"], costs, t, r["slots"], r["events"], flags=flags) == 0


@pytest.mark.parametrize("profile", ["A30", "A100", "H100"])
def test_switch_cost_invariants(O, profile):
    """Zero reconfiguration: the variant equals the literal reading exactly; A30 (no two-size
    node): equal with costs too; with costs: feasible under the variant's validator, and
    non-vacuous (some outputs re-create the {S0..S3} instance)."""
    costs = inputs.reconfig_costs(profile)
    zero = inputs.reconfig_costs(profile, zero=True)
    switched = 0
    for t in list(inputs.synthetic(profile, 16, 30, 61)) + list(inputs.monotone_ties(profile, 12, 20, 62)):
        a = O.far(profile, zero, t)
        b = O.far(profile, zero, t, flags=O.SWITCH_COST)
        assert a["result"] == b["result"] and (a["slots"] == b["slots"]).all()
        r = O.far(profile, costs, t, flags=O.SWITCH_COST)
        assert O.validate(profile, costs, t, r["slots"], r["events"], flags=O.SWITCH_COST) == 0
        if profile == "A30":
            d = O.far(profile, costs, t)
            assert d["result"] == r["result"] and (d["slots"] == r["slots"]).all()
        ncreate1 = sum(1 for e in r["events"] if e["kind"] == 0 and e["node"] == 1)
        switched += ncreate1 > 1
        if ncreate1 > 1:  # the literal validator rejects a re-created node; dropping the switch is caught
            assert O.validate(profile, costs, t, r["slots"], r["events"]) > 0
            keep = [e for e in r["events"] if not (e["node"] == 1 and e["kind"] == 1 and e["start"] < max(
                x["start"] for x in r["events"] if x["node"] == 1))]
            assert O.validate(profile, costs, t, r["slots"], np.array(keep, r["events"].dtype),
                              flags=O.SWITCH_COST) > 0
    if profile != "A30":
        assert switched > 0


@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_int64_domain_scaling(O, profile):
    """The oracle's domain is all int32 times (int64 arithmetic).  Pinned by scale invariance: with
    zero reconfiguration every quantity FAR compares (work s*t, makespans, |2t - m|, |2D - m|) is
    homogeneous of degree 1 in the times, so FAR(c*t) = c*FAR(t) with the same allocation, nodes
    and moves, and starts scaled by c.  c = 2^25 puts every instance beyond the kernel's range
    (sum_i max_s t_i(s) >= 2^29, include/far.h "Integer range")."""
    c = 1 << 25
    for t in list(inputs.synthetic(profile, 9, 6, 41) % 63 + 1) + list(inputs.small_ties(profile, 9, 6, 42)):
        t = np.asarray(t, np.int32)
        assert int(t.max(axis=1).sum()) * c >= 1 << 29
        a = O.far(profile, None, t)
        b = O.far(profile, None, (t.astype(np.int64) * c).astype(np.int32))
        ra, rb = a["result"], b["result"]
        assert rb["makespan"] == c * ra["makespan"]
        assert rb["makespan_phase2"] == c * ra["makespan_phase2"]
        for k in ("alloc_index", "family_size", "moves", "swaps", "evals", "iterations", "reverted", "events"):
            assert rb[k] == ra[k], k
        assert (b["slots"]["node"] == a["slots"]["node"]).all()
        assert (b["slots"]["start"] == c * a["slots"]["start"]).all()


def test_parallel_wrappers_agree_with_sequential(O):
    """The process-pool fan-outs the full-size GPU parity tests use return exactly the sequential
    oracle's makespans / reports (and, with the schedule check, flag a single corrupted slot)."""
    from paper_2507_13601_b200 import inputs
    w = inputs.WORKLOADS["M3"]
    tab = w.table(count=130)
    ms, res = O.far_many(w.profile, w.costs(), tab)
    pm, pr = O.far_many_parallel(w.profile, w.costs(), tab, workers=2)
    assert (pm == ms).all() and (pr == res).all()
    sl = np.zeros((len(tab), tab.shape[1]), O.SLOT_DT)
    for i in range(len(tab)):
        sl[i] = O.far(w.profile, w.costs(), tab[i])["slots"]
    cm, cr, nbad, first = O.far_many_parallel_check(w.profile, w.costs(), tab, sl, workers=2)
    assert (cm == ms).all() and nbad == 0 and first == -1
    sl[77, 3]["start"] += 1
    assert O.far_many_parallel_check(w.profile, w.costs(), tab, sl, workers=2)[2:] == (1, 77)
