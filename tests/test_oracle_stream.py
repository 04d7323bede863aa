"""Oracle pins for the §4 multi-batch fold under DESIGN.md §9's readings.
Parity of this part is pinned by invariants (the paper gives no worked example)."""
import numpy as np
import pytest

from paper_2507_13601_b200 import inputs


def seam(O, profile, tail, first):
    return O.lib().orc_seam_offset_simple(O.pid(profile), np.asarray(tail, np.int64).ctypes.data_as(O.C.c_void_p),
                                          np.asarray(first, np.int64).ctypes.data_as(O.C.c_void_p))


def test_seam_offset_spec_examples(O):
    # SPEC.md:348-350 (DERIVED there from P:655 "try to start B_k after B_{k-1} slice by slice")
    assert seam(O, "A30", [10, 4, 4, 4], [0, 0, 0, 0]) == 10
    assert seam(O, "A30", [10, 4, 4, 4], [6, 0, 0, 0]) == 4
    assert seam(O, "A30", [10, 4, 0, 0], [-1, -1, 0, 0]) == 0      # disjoint slices fully overlap
    assert seam(O, "A100", [5] * 7, [0, 1, 2, 3, 4, 5, 6]) == 5


@pytest.mark.parametrize("profile", ["A30", "A100", "H100"])
@pytest.mark.parametrize("n", [4, 10, 23])
def test_stream_feasible_and_ordered(O, profile, n):
    for seed, costs in ((4, inputs.reconfig_costs(profile)), (9, inputs.reconfig_costs(profile, zero=True))):
        tab = inputs.synthetic(profile, n, 24, seed)
        r = O.stream(profile, costs, tab)
        assert r["violations"] == 0                                   # constraints 1-3 across batches
        offs = r["offsets"]
        assert offs[0] == 0 and (np.diff(offs) >= 0).all()             # offsets non-decreasing (R23)
        assert (r["seam"][:, 0] == np.arange(24) % 2).all()            # odd batches reversed (R21)
        assert (r["seam"][0::2, 1:3] == 0).all()                       # seam ops only on reversed batches
        # every batch of the stream is a FAR schedule of its batch (phases 1-3 reported per batch)
        for k in (0, 5):
            single = O.far(profile, costs, tab[k])["result"]
            assert r["results"][k]["makespan"] == single["makespan"]


def test_stream_single_batch_equals_far(O):
    for profile in ("A30", "A100"):
        costs = inputs.reconfig_costs(profile)
        tab = inputs.synthetic(profile, 12, 1, 3)
        r = O.stream(profile, costs, tab)
        assert r["makespan"] == r["trivial"] == O.far(profile, costs, tab[0])["result"]["makespan"]


def test_reversal_is_a_mirror_without_reconfiguration(O):
    # with zero reconfiguration the reversed schedule is the exact time mirror
    for profile in ("A30", "A100"):
        zero = inputs.reconfig_costs(profile, zero=True)
        t = inputs.synthetic(profile, 9, 1, 21)[0]
        tab = np.stack([t, t])
        r = O.stream(profile, zero, tab, max_iterations=0)
        f = O.far(profile, zero, t, max_iterations=0)
        E = f["result"]["makespan"]
        d = np.array([t[j, inputs.SIZES[profile].index(s)] for j, s in enumerate(f["slots"]["size_used"])])
        assert (r["slots"][0]["start"] == f["slots"]["start"]).all()
        assert (r["slots"][1]["start"] == E - (f["slots"]["start"] + d)).all()
        assert (r["slots"][1]["node"] == f["slots"]["node"]).all()


def test_offset_never_later_than_trivial_start(O):
    # the trivial start (after all previous activity) is always feasible, so the
    # least feasible seam offset can only be earlier
    for profile in ("A30", "A100"):
        costs = inputs.reconfig_costs(profile)
        tab = inputs.synthetic(profile, 10, 16, 77)
        r = O.stream(profile, costs, tab)
        starts = r["offsets"]
        for k in range(1, 16):
            ends = []
            for q in range(k):
                d = np.array([tab[q][j, inputs.SIZES[profile].index(s)]
                              for j, s in enumerate(r["slots"][q]["size_used"])])
                ends.append(starts[q] + (r["slots"][q]["start"] + d).max())
            # all previous tasks end before the trivial start; the smart offset may start earlier
            assert starts[k] <= max(ends) + 2 * 26 * 240


@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_seam_offset_is_least_feasible(O, profile):
    """R23 defines O_k as the LEAST offset >= max(O_{k-1}, 0) for which B_k's timeline is feasible
    after the placed batches.  Pinned independently through the stream validator (constraints 1-3
    across batches, lifecycles): placing B_k one tick earlier must violate something, and placing
    it at O_k must not (checked wherever O_k is above its lower clamp)."""
    checked = 0
    for seed, costs in ((5, inputs.reconfig_costs(profile)), (6, inputs.reconfig_costs(profile, zero=True)),
                        (7, inputs.reconfig_costs(profile))):
        tab = inputs.synthetic(profile, 8, 10, seed)
        r = O.stream(profile, costs, tab)
        offs = r["offsets"]
        for k in range(1, len(tab)):
            o_k, v0 = O.stream_probe(profile, costs, tab, k, 0)
            assert o_k == offs[k] and v0 == 0
            if offs[k] > max(offs[k - 1], 0):
                _, v1 = O.stream_probe(profile, costs, tab, k, 1)
                assert v1 > 0, f"seed {seed} batch {k}: O_k - 1 = {offs[k] - 1} is feasible"
                checked += 1
    assert checked >= 5


GOLD = __import__("json").load(open(__import__("os").path.join(__import__("os").path.dirname(__file__),
                                                             "golden", "spec_traces.json")))


@pytest.mark.parametrize("case", GOLD["stream_seam"], ids=lambda c: c["kind"])
def test_seam_refine_hand_traces(O, case):
    """R24 seam move / swap and R25 trivial concatenation pinned by hand traces (golden trace text)."""
    prof = case["profile"]
    zero = inputs.reconfig_costs(prof, zero=True)
    tab = np.asarray(case["times"], np.int32)
    r = O.stream(prof, zero, tab)
    assert r["offsets"].tolist() == case["offsets"]
    assert (r["makespan"], r["trivial"]) == (case["makespan"], case["trivial"])
    assert r["seam"].tolist() == case["seam"]
    assert [r["slots"][b]["node"].tolist() for b in range(len(tab))] == case["nodes"]
    assert [r["slots"][b]["start"].tolist() for b in range(len(tab))] == case["starts"]
    assert r["violations"] == 0
    rn = O.stream(prof, zero, tab, flags=O.NO_SEAM_MOVES)
    assert rn["offsets"].tolist() == case["no_seam_moves"]["offsets"]
    assert rn["makespan"] == case["no_seam_moves"]["makespan"]
    assert (rn["seam"][:, 1:3] == 0).all()


@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_seam_ops_never_end_later(O, profile):
    """Per-seam invariant of R24's keep-best rule: on the same placed state, batch k with seam
    operations ends (O_k + E_k) no later than without them.  Checked on 2-batch streams, where
    the placed state (batch 0) is the same with and without FAR_NO_SEAM_MOVES."""
    fired = 0
    for seed, costs in ((31, inputs.reconfig_costs(profile)), (32, inputs.reconfig_costs(profile, zero=True))):
        for n in (3, 6, 11):
            tab = inputs.synthetic(profile, n, 40, seed + n).reshape(20, 2, n, -1)
            for pair in tab:
                a = O.stream(profile, costs, pair, ends=True)
                b = O.stream(profile, costs, pair, flags=O.NO_SEAM_MOVES, ends=True)
                assert a["ends"][0] == b["ends"][0]
                assert a["ends"][1] <= b["ends"][1]
                if a["seam"][1, 1] + a["seam"][1, 2]:
                    fired += 1
                    assert a["ends"][1] < b["ends"][1]  # an accepted seam op strictly shortens B_k
    assert fired > 0
