"""GPU parity of multi-target FAR (one tree per MIG GPU, all roots at
time 0) -- far_create_multi + the forest kernel against the oracle's forest, bit-exact on every
field and every task slot."""
import numpy as np
import pytest

from paper_2507_13601_b200 import far, inputs
from test_gpu_parity import check_against_oracle, run_gpu

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch, torch.device("cuda:0")


@pytest.mark.parametrize("prof,n", [("A30x2", 8), ("A30x2", 33), ("A30x3", 20), ("A100x2", 16), ("A100x2", 64),
                                    ("H100x4", 40), ("A100x8", 128), ("A30x8", 256), ("A100x2", 0),
                                    ("A100x3", 1), ("A30x2", 7)])
def test_forest_bitexact(O, torch_dev, prof, n):
    base = prof.split("x")[0]
    costs = inputs.reconfig_costs(base)
    count = 60 if n >= 128 else 200
    tab = inputs.synthetic(base, n, count, 500 + n)
    for flags in (0, far.EXHAUSTIVE, far.NO_GUARD, far.ZERO_RECONFIG, far.NO_REFINE, far.BEST_IMPROVEMENT):
        ms, slots, res = run_gpu(torch_dev, prof, costs, tab, flags=flags)
        check_against_oracle(O, prof, costs, tab, ms, slots, res, flags=flags, full=n <= 64)


@pytest.mark.parametrize("prof,gen", [("A30x2", "ties"), ("A100x2", "ties"), ("A100x2", "uniform"),
                                      ("A100x4", "monoties")])
def test_forest_ties_and_variants(O, torch_dev, prof, gen):
    base = prof.split("x")[0]
    costs = inputs.reconfig_costs(base)
    n = 24
    tab = {"ties": inputs.small_ties, "uniform": inputs.uniform_random,
           "monoties": inputs.monotone_ties}[gen](base, n, 200, 41)
    for flags in (0, far.NONEMPTY_ALT, far.GROW_TIES, far.GROW_TIES | far.EXHAUSTIVE, far.BEST_IMPROVEMENT,
                  far.BEST_IMPROVEMENT | far.ZERO_RECONFIG):
        ms, slots, res = run_gpu(torch_dev, prof, costs, tab, flags=flags)
        check_against_oracle(O, prof, costs, tab, ms, slots, res, flags=flags)
    for flags in (0, far.BEST_IMPROVEMENT):
        for kw in ({"max_iterations": 1}, {"min_improvement_ppm": 30000}):
            ms, slots, res = run_gpu(torch_dev, prof, costs, tab, flags=flags, **kw)
            check_against_oracle(O, prof, costs, tab, ms, slots, res, flags=flags,
                                 max_iterations=kw.get("max_iterations", 100),
                                 ppm=kw.get("min_improvement_ppm", 0), full=False)


def test_forest_more_gpus_help(O, torch_dev):
    """Non-vacuous: on the same batches, more MIG GPUs give shorter FAR schedules on average, and
    the g-GPU schedules differ from the single-GPU ones."""
    tab = inputs.synthetic("A100", 32, 300, 77)
    costs = inputs.reconfig_costs("A100")
    m1 = run_gpu(torch_dev, "A100", costs, tab)[0]
    m2 = run_gpu(torch_dev, "A100x2", costs, tab)[0]
    m4 = run_gpu(torch_dev, "A100x4", costs, tab)[0]
    assert m4.mean() < m2.mean() < m1.mean()


def test_forest_host_paths(O, torch_dev):
    for prof in ("A30x2", "A100x3"):
        base = prof.split("x")[0]
        costs = inputs.reconfig_costs(base)
        F = far.Far(prof, costs)
        assert F.gpus == int(prof.split("x")[1]) and F.nnodes == len(O.nodes(prof)[0])
        lo, hi, par = F.node_table()
        olo, ohi, opar = O.nodes(prof)
        assert (lo == olo).all() and (hi == ohi).all() and (par == opar).all()
        for t in inputs.synthetic(base, 19, 30, 58):
            s, r = F.schedule_batch(t)
            o = O.far(prof, costs, t, flags=O.NO_REFINE)
            assert (s["node"] == o["slots"]["node"]).all() and (s["start"] == o["slots"]["start"]).all()
            assert r["makespan"] == o["result"]["makespan"] and r["alloc_index"] == o["result"]["alloc_index"]
            s2, r2 = F.local_search(t, s, makespan_phase2=int(r["makespan"]))
            oslots = np.zeros(len(s), O.SLOT_DT)
            oslots["node"], oslots["size_used"], oslots["start"] = s["node"], s["size_used"], s["start"]
            q = O.refine(prof, costs, t, oslots, int(r["makespan"]))
            for k in ("makespan", "moves", "swaps", "evals", "iterations", "reverted"):
                assert r2[k] == q["result"][k], k
            assert (s2["node"] == q["slots"]["node"]).all() and (s2["start"] == q["slots"]["start"]).all()
            s3, r3 = F.local_search(t, s, makespan_phase2=int(r["makespan"]), flags=far.BEST_IMPROVEMENT)
            q3 = O.refine(prof, costs, t, oslots, int(r["makespan"]), flags=O.BEST_IMPROVEMENT)
            for k in ("makespan", "moves", "swaps", "evals", "iterations", "reverted"):
                assert r3[k] == q3["result"][k], k
            assert (s3["node"] == q3["slots"]["node"]).all() and (s3["start"] == q3["slots"]["start"]).all()
        tab = np.ascontiguousarray(inputs.synthetic(base, 21, 500, 59))
        ms_h, sd_h, rs_h = F.solve_many_host(tab)
        oms, _ = O.far_many(prof, costs, tab)
        assert (ms_h == oms).all()


def test_forest_errors(torch_dev):
    torch, dev = torch_dev
    F = far.Far("A100x2")
    d = torch.ones((2, 257, 5), dtype=torch.int32, device=dev)
    with pytest.raises(far.FarError):
        F.solve_many(d)
    d = torch.ones((2, 8, 5), dtype=torch.int32, device=dev)
    with pytest.raises(far.FarError):
        F.concat_streams(d.reshape(1, 2, 8, 5))
    with pytest.raises(far.FarError):
        far.Far("A100x9")


@pytest.mark.parametrize("prof,n,count", [("A30x2", 16, 100), ("A100x2", 24, 100), ("A100x4", 40, 60),
                                          ("H100x3", 12, 100), ("A30x8", 64, 30), ("A100x8", 128, 12)])
def test_forest_events_match_oracle(O, torch_dev, prof, n, count):
    """far_schedule_events / far_validate_schedules on multi-target contexts (NEXT-2 x NEXT-4): the
    forest replay's creates and the destroys issued while tasks remain equal the oracle's event list
    of the same FAR output, the replay reproduces the makespan, and every output is feasible for both
    validators."""
    import test_gpu_check as TC
    base = prof.split("x")[0]
    costs = inputs.reconfig_costs(base)
    tab = inputs.synthetic(base, n, count, 700 + n)
    for flags in (0, far.NO_REFINE, far.ZERO_RECONFIG):
        F, d, sd, ms, slots, evs, nev, ems, viol = TC.solve_and_events(torch_dev, prof, costs, tab, flags=flags)
        assert (ems == ms).all(), "the replay of a FAR output reproduces its makespan (fixpoint)"
        assert (viol == 0).all(), f"infeasible outputs at {np.nonzero(viol)[0][:10]}"
        for i in range(count):
            o = O.far(prof, costs, tab[i], flags=flags & (O.NO_REFINE | O.ZERO_RECONFIG))
            assert TC.ordered(evs[i]) == TC.ordered(o["events"]), f"{prof} flags {flags}: events differ, instance {i}"
            oc = inputs.reconfig_costs(base, zero=True) if flags & far.ZERO_RECONFIG else costs
            assert O.validate(prof, oc, tab[i], TC.to_oracle_slots(slots[i]), TC.to_oracle_events(evs[i])) == 0


@pytest.mark.parametrize("prof", ["A30x2", "A100x3"])
def test_forest_validator_counts_match_oracle(O, torch_dev, prof):
    """Violation counts of corrupted multi-target schedules and events equal orc_validate's."""
    import test_gpu_check as TC
    torch, dev = torch_dev
    base = prof.split("x")[0]
    costs = inputs.reconfig_costs(base)
    tab = inputs.synthetic(base, 14, 300, 41)
    F, d, sd, ms, slots, evs, nev, ems, viol = TC.solve_and_events(torch_dev, prof, costs, tab)
    lo, hi, _ = F.node_table()
    rng = np.random.default_rng(6)
    cap = 2 * F.nnodes
    S = np.zeros((tab.shape[0], tab.shape[1]), far.SLOT_DT)
    E = np.zeros((tab.shape[0], cap), far.EVENT_DT)
    NE = np.zeros(tab.shape[0], np.int32)
    for i in range(tab.shape[0]):
        s, e = slots[i], evs[i]
        for _ in range(rng.integers(1, 3)):
            s, e = TC.perturb(rng, prof, s, e, tab[i], lo, hi)
        e = e[:cap]
        S[i], E[i, :len(e)], NE[i] = s, e, len(e)
    dS = torch.from_numpy(S.view(np.uint8).reshape(tab.shape[0], tab.shape[1], 8)).to(dev)
    dE = torch.from_numpy(E.view(np.uint8).reshape(tab.shape[0], cap, 16)).to(dev)
    dN = torch.from_numpy(NE).to(dev)
    v = F.validate_schedules(d, dS, dE, dN).cpu().numpy()
    want = np.array([O.validate(prof, costs, tab[i], TC.to_oracle_slots(S[i]), TC.to_oracle_events(E[i, :NE[i]]))
                     for i in range(tab.shape[0])])
    assert (v == want).all(), f"mismatch at {np.nonzero(v != want)[0][:10]}: gpu {v[v != want][:5]} oracle {want[v != want][:5]}"
    assert (want > 0).mean() > 0.5
