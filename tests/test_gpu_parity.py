"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by
element, on seeded inputs.  Integer work -> bit-exact on every field."""
import numpy as np
import pytest

from paper_2507_13601_b200 import far, inputs

pytestmark = pytest.mark.gpu

FIELDS = ("makespan", "makespan_phase2", "alloc_index", "family_size", "moves", "swaps", "iterations", "reverted",
          "evals")


@pytest.fixture(scope="module")
def torch_dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch, torch.device("cuda:0")


def _solve(torch_dev, profile, costs, tab, **kw):
    torch, dev = torch_dev
    F = far.Far(profile, costs)
    d = torch.from_numpy(np.ascontiguousarray(tab)).to(dev)
    ms, sd, rs = F.solve_many(d, **kw)
    torch.cuda.synchronize()
    F.sync()
    return ms.cpu().numpy(), far.slots_np(sd), far.results_np(rs)


def run_gpu(torch_dev, profile, costs, tab, **kw):
    """Batches below 256 instances take the fused one-launch kernel (latency); they are solved a
    second time through the pipelined chain (FAR_PIPELINE_ALWAYS) and both must agree bit for bit."""
    import os
    out = _solve(torch_dev, profile, costs, tab, **kw)
    if len(tab) < 256 and "FAR_PIPELINE_ALWAYS" not in os.environ:
        os.environ["FAR_PIPELINE_ALWAYS"] = "1"
        try:
            alt = _solve(torch_dev, profile, costs, tab, **kw)
        finally:
            del os.environ["FAR_PIPELINE_ALWAYS"]
        assert (alt[0] == out[0]).all()
        if out[1] is not None:
            assert (alt[1] == out[1]).all()
        if out[2] is not None:
            # Alg. 1 pop counts depend on which members each path simulates; the rest is identical
            for k in out[2].dtype.names:
                if k != "events":
                    assert (alt[2][k] == out[2][k]).all(), k
    return out


def check_against_oracle(O, profile, costs, tab, ms, slots, res, flags=0, max_iterations=100, ppm=0, full=True):
    oflags = flags & (O.NO_REFINE | O.NO_GUARD | O.ZERO_RECONFIG | O.NONEMPTY_ALT | O.GROW_TIES | O.BEST_IMPROVEMENT |
                      O.SWITCH_COST)
    oms, ores = O.far_many(profile, costs, tab, max_iterations=max_iterations, min_improvement_ppm=ppm, flags=oflags)
    bad = np.nonzero(ms != oms)[0]
    assert len(bad) == 0, f"makespan mismatch at {bad[:10]}: gpu {ms[bad[:5]]} oracle {oms[bad[:5]]}"
    for k in FIELDS:
        assert (res[k] == ores[k]).all(), f"{k} mismatch at {np.nonzero(res[k] != ores[k])[0][:10]}"
    # Alg. 1 pops: all members with FAR_EXHAUSTIVE, otherwise only the members not skipped
    if flags & far.EXHAUSTIVE:
        assert (res["events"] == ores["events"]).all()
    else:
        assert (res["events"] <= ores["events"]).all() and (res["events"] > 0).sum() == (ores["events"] > 0).sum()
    if full and slots is not None:
        for i in range(tab.shape[0]):
            o = O.far(profile, costs, tab[i], max_iterations=max_iterations, min_improvement_ppm=ppm, flags=oflags)
            os_ = o["slots"]
            assert (slots[i]["node"] == os_["node"]).all(), f"node mismatch instance {i}"
            assert (slots[i]["size_used"] == os_["size_used"]).all(), f"size_used mismatch instance {i}"
            assert (slots[i]["start"] == os_["start"]).all(), f"start mismatch instance {i}"


@pytest.mark.parametrize("wname,count", [("M1", 2000), ("M2", 2000), ("M3", 1000), ("M5", 300)])
def test_workload_samples_bitexact(O, torch_dev, wname, count):
    w = inputs.WORKLOADS[wname]
    tab = w.table(count=count)
    for flags in (0, far.EXHAUSTIVE):
        ms, slots, res = run_gpu(torch_dev, w.profile, w.costs(), tab, flags=flags)
        check_against_oracle(O, w.profile, w.costs(), tab, ms, slots, res, flags=flags, full=True)


@pytest.mark.parametrize("profile", ["A30", "A100", "H100"])
@pytest.mark.parametrize("n", [0, 1, 2, 7, 31, 32, 33, 64, 65])
def test_ragged_sizes(O, torch_dev, profile, n):
    costs = inputs.reconfig_costs(profile)
    tab = inputs.synthetic(profile, n, 97, 1000 + n)
    ms, slots, res = run_gpu(torch_dev, profile, costs, tab)
    check_against_oracle(O, profile, costs, tab, ms, slots, res)


@pytest.mark.parametrize("profile", ["A30", "A100"])
@pytest.mark.parametrize("gen", ["ties", "monoties", "uniform", "narrow", "poor", "good"])
def test_tie_and_nonmonotone_inputs(O, torch_dev, profile, gen):
    n = 24
    if gen == "ties":
        tab = inputs.small_ties(profile, n, 300, 5)
    elif gen == "monoties":
        tab = inputs.monotone_ties(profile, n, 300, 15)
    elif gen == "uniform":
        tab = inputs.uniform_random(profile, n, 300, 6)       # non-monotone runtimes
    elif gen == "narrow":
        tab = inputs.synthetic(profile, n, 300, 7, times="narrow")
    else:
        tab = inputs.synthetic(profile, n, 300, 8, scaling=gen)
    for costs in (inputs.reconfig_costs(profile), inputs.reconfig_costs(profile, zero=True)):
        ms, slots, res = run_gpu(torch_dev, profile, costs, tab)
        check_against_oracle(O, profile, costs, tab, ms, slots, res)


@pytest.mark.parametrize("flags,max_it,ppm", [(far.EXHAUSTIVE, 100, 0), (far.EXHAUSTIVE | far.NO_REFINE, 100, 0),
                                               (far.NO_REFINE, 100, 0), (far.NO_GUARD, 100, 0),
                                               (far.ZERO_RECONFIG, 100, 0), (0, 0, 0), (0, 1, 0), (0, 3, 0),
                                               (0, 100, 20000)])
def test_options(O, torch_dev, flags, max_it, ppm):
    profile = "A100"
    costs = inputs.reconfig_costs(profile)
    tab = inputs.synthetic(profile, 20, 400, 21)
    ms, slots, res = run_gpu(torch_dev, profile, costs, tab, flags=flags, max_iterations=max_it,
                             min_improvement_ppm=ppm)
    check_against_oracle(O, profile, costs, tab, ms, slots, res, flags=flags, max_iterations=max_it, ppm=ppm)


@pytest.mark.parametrize("n", [128, 256, 257, 600, 1023, 1024])
def test_large_n(O, torch_dev, n):
    profile = "A100"
    costs = inputs.reconfig_costs(profile)
    big = n > 512
    tab = inputs.synthetic(profile, n, 24 if not big else 3, 31, times="narrow" if big else "wide")
    if big:
        tab = np.minimum(tab, 900)  # keep the makespan bound < 2^29
    ms, slots, res = run_gpu(torch_dev, profile, costs, tab)
    check_against_oracle(O, profile, costs, tab, ms, slots, res)


# The pipelined solver has three H6/H7 implementations: one thread per instance (n <= 256),
# one warp per instance (the debug switch below, and 256 < n <= 1023), and the fused kernel
# (FAR_FUSED_PHASE2; also the overflow pass and n = 1024).  All must agree with the oracle.
@pytest.mark.parametrize("switch", [None, "FAR_DEBUG_WARP_FINISH", "FAR_FUSED_PHASE2"])
@pytest.mark.parametrize("wname,gen", [("M5", "wide"), ("M3", "wide"), ("A30", "ties"), ("A100", "monoties")])
def test_finish_paths_agree(O, torch_dev, monkeypatch, switch, wname, gen):
    if switch:
        monkeypatch.setenv(switch, "1")
    if wname in ("M5", "M3"):
        w = inputs.WORKLOADS[wname]
        profile, costs, tab = w.profile, w.costs(), w.table(count=200)
    elif gen == "ties":
        profile = wname
        costs, tab = inputs.reconfig_costs(profile), inputs.small_ties(profile, 40, 200, 8)
    else:
        profile = wname
        costs, tab = inputs.reconfig_costs(profile), inputs.monotone_ties(profile, 40, 200, 9)
    for flags in (0, far.NO_GUARD, far.NONEMPTY_ALT):
        ms, slots, res = run_gpu(torch_dev, profile, costs, tab, flags=flags)
        check_against_oracle(O, profile, costs, tab, ms, slots, res, flags=flags)


@pytest.mark.parametrize("profile,gen", [("A30", "ties"), ("A100", "ties"), ("A100", "monoties"), ("H100", "mixed")])
def test_grow_ties_variant(O, torch_dev, profile, gen):
    # the NEXT-3 reading variant FAR_GROW_TIES (phase 1 grows all tied longest tasks)
    # against the oracle, and non-vacuous on tie-heavy inputs
    costs = inputs.reconfig_costs(profile)
    if gen == "ties":
        tab = inputs.small_ties(profile, 20, 300, 44)
    elif gen == "monoties":
        tab = inputs.monotone_ties(profile, 24, 300, 45)
    else:
        tab = inputs.synthetic(profile, 32, 300, 46)
    ms0, _, r0 = run_gpu(torch_dev, profile, costs, tab)
    for flags in (far.GROW_TIES, far.GROW_TIES | far.EXHAUSTIVE, far.GROW_TIES | far.NONEMPTY_ALT):
        ms1, s1, r1 = run_gpu(torch_dev, profile, costs, tab, flags=flags)
        check_against_oracle(O, profile, costs, tab, ms1, s1, r1, flags=flags)
    if gen != "mixed":
        assert (r0["family_size"] != r1["family_size"]).any()


@pytest.mark.parametrize("profile,n", [("A100", 10), ("A100", 16), ("A30", 8)])
def test_nonempty_alt_variant(O, torch_dev, profile, n):
    # the NEXT-3 reading variant (FAR_NONEMPTY_ALT) against the oracle on small batches, where
    # empty same-size nodes are common, and non-vacuous: it changes some outcomes
    costs = inputs.reconfig_costs(profile)
    tab = inputs.synthetic(profile, n, 300, 41)
    ms0, _, r0 = run_gpu(torch_dev, profile, costs, tab)
    ms1, s1, r1 = run_gpu(torch_dev, profile, costs, tab, flags=far.NONEMPTY_ALT)
    check_against_oracle(O, profile, costs, tab, ms1, s1, r1, flags=far.NONEMPTY_ALT)
    assert (r0["evals"] != r1["evals"]).any() and (ms0 != ms1).any()


def test_input_errors_flagged(torch_dev):
    torch, dev = torch_dev
    tab = inputs.synthetic("A30", 5, 4, 3)
    tab[1, 2, 1] = 0                      # t < 1
    tab[2, :, :] = 1 << 29                # makespan bound
    F = far.Far("A30")
    ms, sd, rs = F.solve_many(torch.from_numpy(tab).to(dev))
    torch.cuda.synchronize()
    r = far.results_np(rs)
    assert ms.cpu().numpy().tolist()[1:3] == [-1, -1]
    assert r["status"].tolist() == [0, 3, 3, 0]
    with pytest.raises(far.FarError) as e:
        F.sync()
    assert e.value.status == 3
    F.sync()  # flag cleared


def test_kernel_range_is_narrower_than_the_oracle(O, torch_dev):
    """The kernel's int32 range (include/far.h "Integer range": sum_i max_s t_i(s) + costs < 2^29)
    is its own contract: inputs beyond it are still solved by the int64 oracle, and the kernel
    flags them FAR_E_BAD_TIME instead of returning a wrong schedule."""
    torch, dev = torch_dev
    for profile in ("A30", "A100"):
        tab = (inputs.synthetic(profile, 9, 4, 41) % 63 + 1).astype(np.int64) << 25
        tab = tab.astype(np.int32)
        for t in tab:
            assert O.far(profile, None, t)["result"]["makespan"] > 0
        F = far.Far(profile, inputs.reconfig_costs(profile, zero=True))
        ms, sd, rs = F.solve_many(torch.from_numpy(tab).to(dev))
        torch.cuda.synchronize()
        assert (ms.cpu().numpy() == -1).all()
        assert (far.results_np(rs)["status"] == 3).all()
        with pytest.raises(far.FarError) as e:
            F.sync()
        assert e.value.status == 3


def test_schedule_batch_and_local_search(O, torch_dev):
    for profile in ("A30", "A100", "H100"):
        costs = inputs.reconfig_costs(profile)
        F = far.Far(profile, costs)
        for t in inputs.synthetic(profile, 19, 60, 55):
            s, r = F.schedule_batch(t)
            o = O.far(profile, costs, t, flags=O.NO_REFINE)
            assert (s["node"] == o["slots"]["node"]).all() and (s["start"] == o["slots"]["start"]).all()
            assert r["makespan"] == o["result"]["makespan"] and r["alloc_index"] == o["result"]["alloc_index"]
            # phase 3 on the phase-2 schedule == the oracle's refine
            s2, r2 = F.local_search(t, s, makespan_phase2=int(r["makespan"]))
            oslots = np.zeros(len(s), O.SLOT_DT)
            oslots["node"], oslots["size_used"], oslots["start"] = s["node"], s["size_used"], s["start"]
            q = O.refine(profile, costs, t, oslots, int(r["makespan"]))
            assert r2["makespan"] == q["result"]["makespan"]
            for k in ("moves", "swaps", "evals", "iterations", "reverted"):
                assert r2[k] == q["result"][k], k
            assert (s2["node"] == q["slots"]["node"]).all() and (s2["start"] == q["slots"]["start"]).all()
            # and it equals the full pipeline
            full = O.far(profile, costs, t)
            assert r2["makespan"] == full["result"]["makespan"]


@pytest.mark.parametrize("chunk_mb", [None, "1"])
def test_host_pipeline_matches_device(torch_dev, monkeypatch, chunk_mb):
    """far_solve_many_host (H2D / chain / D2H over two streams) == far_solve_many; with 1-MB chunks
    the 5000 instances cross ~17 chunks alternating between the streams and the workspaces."""
    if chunk_mb:
        monkeypatch.setenv("FAR_HOST_CHUNK_MB", chunk_mb)
    w = inputs.WORKLOADS["M3"]
    tab = w.table(count=5000)
    ms, slots, res = run_gpu(torch_dev, w.profile, w.costs(), tab)
    F = far.Far(w.profile, w.costs())
    hms, hsl, hres = F.solve_many_host(tab)
    assert (hms == ms).all() and (hsl["start"] == slots["start"]).all() and (hsl["node"] == slots["node"]).all()
    for k in FIELDS:
        assert (hres[k] == res[k]).all(), k


def test_full_size_m3_parity(O, torch_dev):
    """BASELINE configs[2]: all 100k A100 x n=32 instances, every field bit-exact (makespans and
    reports on all instances; oracle fanned out over the host cores)."""
    w = inputs.WORKLOADS["M3"]
    tab = w.table(parallel=True)
    ms, slots, res = run_gpu(torch_dev, w.profile, w.costs(), tab)
    oms, ores = O.far_many_parallel(w.profile, w.costs(), tab)
    assert (ms == oms).all()
    for k in FIELDS:
        assert (res[k] == ores[k]).all(), k
    rng = np.random.default_rng(0)
    for i in rng.choice(len(tab), 200, replace=False):
        o = O.far(w.profile, w.costs(), tab[i])
        assert (slots[i]["node"] == o["slots"]["node"]).all() and (slots[i]["start"] == o["slots"]["start"]).all()


def test_full_size_m5_sampled(O, torch_dev):
    """BASELINE configs[4] at full size in the bench's launch configuration (1M x n=128 on one GPU):
    sampled instances bit-exact against the oracle; properties on every instance."""
    torch, dev = torch_dev
    w = inputs.WORKLOADS["M5"]
    tab = w.table(parallel=True)
    F = far.Far(w.profile, w.costs())
    d = torch.from_numpy(tab).to(dev)
    ms, sd, rs = F.solve_many(d)
    torch.cuda.synchronize()
    F.sync()
    ms = ms.cpu().numpy()
    res = far.results_np(rs)
    del d
    # properties on all 1M: lower bounds, guard, family bound
    t64 = tab.astype(np.int64)
    sizes = np.array(inputs.SIZES[w.profile], np.int64)
    W = (t64 * sizes).min(axis=2).sum(axis=1)
    H = t64.min(axis=2).max(axis=1)
    assert (7 * ms.astype(np.int64) >= W).all() and (ms >= H).all()
    assert (res["makespan"] <= res["makespan_phase2"]).all() and (res["status"] == 0).all()
    assert (res["family_size"] >= 1).all() and (res["family_size"] <= 1 + 128 * 4).all()
    rng = np.random.default_rng(1)
    idx = np.sort(rng.choice(len(tab), 300, replace=False))
    slots = far.slots_np(sd[torch.from_numpy(idx).to(sd.device)])
    oms, ores = O.far_many(w.profile, w.costs(), tab[idx])
    assert (ms[idx] == oms).all()
    for k in FIELDS:
        assert (res[k][idx] == ores[k]).all(), k
    for q, i in enumerate(idx[:40]):
        o = O.far(w.profile, w.costs(), tab[i])
        assert (slots[q]["node"] == o["slots"]["node"]).all() and (slots[q]["start"] == o["slots"]["start"]).all()


def test_local_search_on_other_schedules(O, torch_dev):
    """far_local_search on schedules other than phase 2's (the refined FAR schedule itself, with
    its start order) equals the oracle's Alg. 2 + replay + guard on the same input."""
    for profile in ("A30", "A100"):
        costs = inputs.reconfig_costs(profile)
        F = far.Far(profile, costs)
        for t in inputs.synthetic(profile, 21, 40, 71):
            o = O.far(profile, costs, t)
            s_in = np.zeros(len(t), far.SLOT_DT)
            s_in["node"], s_in["size_used"], s_in["start"] = o["slots"]["node"], o["slots"]["size_used"], o["slots"]["start"]
            ms_in = int(o["result"]["makespan"])
            s2, r2 = F.local_search(t, s_in, makespan_phase2=ms_in)
            q = O.refine(profile, costs, t, o["slots"], ms_in)
            assert r2["makespan"] == q["result"]["makespan"] and r2["reverted"] == q["result"]["reverted"]
            assert (s2["node"] == q["slots"]["node"]).all() and (s2["start"] == q["slots"]["start"]).all()
            assert r2["makespan"] <= ms_in


def test_local_search_rejects_bad_schedules(torch_dev):
    F = far.Far("A30")
    t = inputs.synthetic("A30", 4, 1, 3)[0]
    s, r = F.schedule_batch(t)
    bad = s.copy()
    bad["node"][0] = 9                     # no such tree node
    with pytest.raises(far.FarError) as e:
        F.local_search(t, bad)
    assert e.value.status == 1
    bad = s.copy()
    bad["size_used"][0] = 3                # A30 hosts no size 3
    with pytest.raises(far.FarError) as e:
        F.local_search(t, bad)
    assert e.value.status == 1
    F.sync()


@pytest.mark.parametrize("profile,gen,n", [("A30", "mixed", 8), ("A30", "ties", 20), ("A100", "mixed", 16),
                                           ("A100", "ties", 24), ("A100", "uniform", 33), ("H100", "mixed", 70),
                                           ("A100", "mixed", 128), ("A100", "mixed", 300)])
def test_best_improvement_variant(O, torch_dev, profile, gen, n):
    """The NEXT-3 variant FAR_BEST_IMPROVEMENT (R30: every same-size move and every swap
    pair scored by the resulting makespan, argmin applied) against the oracle, bit-exact on every
    field incl. evals; non-vacuous (it changes some refinements)."""
    costs = inputs.reconfig_costs(profile)
    count = 40 if n >= 128 else 200
    if gen == "ties":
        tab = inputs.small_ties(profile, n, count, 61)
    elif gen == "uniform":
        tab = inputs.uniform_random(profile, n, count, 62)
    else:
        tab = inputs.synthetic(profile, n, count, 63 + n)
    BI = far.BEST_IMPROVEMENT
    _, _, r0 = run_gpu(torch_dev, profile, costs, tab)
    for flags in (BI, BI | far.NO_GUARD, BI | far.ZERO_RECONFIG, BI | far.EXHAUSTIVE | far.GROW_TIES):
        ms, slots, res = run_gpu(torch_dev, profile, costs, tab, flags=flags)
        check_against_oracle(O, profile, costs, tab, ms, slots, res, flags=flags, full=n <= 128)
        if flags == BI:
            assert (res["evals"] != r0["evals"]).any()
    # max_iterations = 1 and a min-improvement threshold
    for kw in ({"max_iterations": 1}, {"min_improvement_ppm": 20000}):
        ms, slots, res = run_gpu(torch_dev, profile, costs, tab, flags=BI, **kw)
        check_against_oracle(O, profile, costs, tab, ms, slots, res, flags=BI,
                             max_iterations=kw.get("max_iterations", 100), ppm=kw.get("min_improvement_ppm", 0),
                             full=False)


def test_best_improvement_local_search(O, torch_dev):
    """far_local_search with FAR_BEST_IMPROVEMENT on phase-2 schedules == the oracle's refine."""
    for profile in ("A30", "A100"):
        costs = inputs.reconfig_costs(profile)
        F = far.Far(profile, costs)
        for t in inputs.synthetic(profile, 18, 40, 57):
            s, r = F.schedule_batch(t)
            s2, r2 = F.local_search(t, s, makespan_phase2=int(r["makespan"]), flags=far.BEST_IMPROVEMENT)
            oslots = np.zeros(len(s), O.SLOT_DT)
            oslots["node"], oslots["size_used"], oslots["start"] = s["node"], s["size_used"], s["start"]
            q = O.refine(profile, costs, t, oslots, int(r["makespan"]), flags=O.BEST_IMPROVEMENT)
            for k in ("makespan", "moves", "swaps", "evals", "iterations", "reverted"):
                assert r2[k] == q["result"][k], k
            assert (s2["node"] == q["slots"]["node"]).all() and (s2["start"] == q["slots"]["start"]).all()


@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_best_improvement_fused_path(O, torch_dev, monkeypatch, profile):
    monkeypatch.setenv("FAR_FUSED_PHASE2", "1")
    costs = inputs.reconfig_costs(profile)
    tab = inputs.synthetic(profile, 40, 100, 64)
    ms, slots, res = run_gpu(torch_dev, profile, costs, tab, flags=far.BEST_IMPROVEMENT)
    check_against_oracle(O, profile, costs, tab, ms, slots, res, flags=far.BEST_IMPROVEMENT)


@pytest.mark.parametrize("n", [128, 511])
def test_grow_ties_many_entries(O, torch_dev, n):
    """Regression (found by tests/test_gpu_fuzz.py seed 151): with FAR_GROW_TIES and dense ties a
    growth step adds one list entry per tied task, so the per-size lists can outgrow the fast
    layout before the family does; such instances must go to the full-layout overflow pass."""
    costs = inputs.reconfig_costs("H100")
    tab = inputs.monotone_ties("H100", n, 6 if n > 256 else 40, 7)
    for flags in (far.GROW_TIES | far.NO_REFINE, far.GROW_TIES):
        ms, slots, res = run_gpu(torch_dev, "H100", costs, tab, flags=flags)
        check_against_oracle(O, "H100", costs, tab, ms, slots, res, flags=flags, full=n <= 128)


@pytest.mark.skipif(bool(__import__("os").environ.get("FAR_SKIP_FULL_M5")), reason="opt-out")
def test_full_size_m5_parity(O, torch_dev):
    """BASELINE configs[4] at full size: all 1M A100 x n=128 instances of the bench workload, the
    makespan, every report field AND every task slot (node, size used, start) of all 1M schedules
    bit-exact (oracle fanned out over the host cores, the schedules compared chunk by chunk inside
    the workers; ~1 min on the 16-core B200 host)."""
    torch, dev = torch_dev
    w = inputs.WORKLOADS["M5"]
    tab = w.table(parallel=True)
    F = far.Far(w.profile, w.costs())
    ms, sd, rs = F.solve_many(torch.from_numpy(tab).to(dev))
    torch.cuda.synchronize()
    F.sync()
    ms, res, slots = ms.cpu().numpy(), far.results_np(rs), far.slots_np(sd)
    del sd
    oms, ores, nbad, first = O.far_many_parallel_check(w.profile, w.costs(), tab, slots)
    assert (ms == oms).all(), f"makespan mismatch at {np.nonzero(ms != oms)[0][:10]}"
    for k in FIELDS:
        assert (res[k] == ores[k]).all(), k
    assert nbad == 0, f"{nbad} schedules differ, first at instance {first}"


@pytest.mark.parametrize("world,rank", [(8, 7), (4, 1)])
def test_strong_scaling_shard_parity(O, torch_dev, world, rank):
    """Config 5 under strong scaling: the shard one rank solves (dist.shard_range(1M, rank, world):
    125k instances at N = 8 -- the members stage's one-to-two-round branch -- and 250k at N = 4),
    generated exactly as bench.py does (counter-based table from the shard's first index), solved
    on the GPU at the shard's size, every makespan, report field and task slot bit-exact."""
    from paper_2507_13601_b200 import dist as fdist
    torch, dev = torch_dev
    w = inputs.WORKLOADS["M5"]
    lo, hi = fdist.shard_range(1_000_000, rank, world)
    tab = inputs.synthetic_parallel(w.profile, w.n, hi - lo, w.seed, scaling=w.scaling, times=w.times, start=lo)
    F = far.Far(w.profile, w.costs())
    ms, sd, rs = F.solve_many(torch.from_numpy(tab).to(dev))
    torch.cuda.synchronize()
    F.sync()
    ms, res, slots = ms.cpu().numpy(), far.results_np(rs), far.slots_np(sd)
    oms, ores, nbad, first = O.far_many_parallel_check(w.profile, w.costs(), tab, slots)
    assert (ms == oms).all(), f"makespan mismatch at {np.nonzero(ms != oms)[0][:10]}"
    for k in FIELDS:
        assert (res[k] == ores[k]).all(), k
    assert nbad == 0, f"{nbad} schedules differ, first at instance {first}"


@pytest.mark.parametrize("profile,gen,n", [("A100", "mixed", 16), ("H100", "mixed", 40), ("A100", "ties", 24),
                                           ("A100", "monoties", 24), ("A30", "mixed", 12), ("A100", "mixed", 300)])
def test_switch_cost_variant(O, torch_dev, profile, gen, n):
    """The NEXT-3 variant FAR_SWITCH_COST (R7: the {S0..S3} node re-created on a 4->3
    switch, instances created / destroyed at their task size) against the oracle; non-vacuous."""
    costs = inputs.reconfig_costs(profile)
    count = 30 if n > 256 else 300
    tab = {"mixed": inputs.synthetic, "ties": inputs.small_ties, "monoties": inputs.monotone_ties}[gen](
        profile, n, count, 90 + n)
    _, _, r0 = run_gpu(torch_dev, profile, costs, tab)
    for flags in (far.SWITCH_COST, far.SWITCH_COST | far.NO_GUARD, far.SWITCH_COST | far.EXHAUSTIVE | far.GROW_TIES,
                  far.SWITCH_COST | far.BEST_IMPROVEMENT, far.SWITCH_COST | far.NO_REFINE):
        ms, slots, res = run_gpu(torch_dev, profile, costs, tab, flags=flags)
        check_against_oracle(O, profile, costs, tab, ms, slots, res, flags=flags, full=n <= 64)
        if flags == far.SWITCH_COST and profile != "A30":
            assert (res["makespan_phase2"] != r0["makespan_phase2"]).any()


def test_switch_cost_local_search_and_forest(O, torch_dev):
    for prof in ("A100", "H100x2"):
        base = prof.split("x")[0]
        costs = inputs.reconfig_costs(base)
        F = far.Far(prof, costs)
        for t in inputs.synthetic(base, 20, 20, 92):
            s, r = F.schedule_batch(t, flags=far.SWITCH_COST)
            o = O.far(prof, costs, t, flags=O.NO_REFINE | O.SWITCH_COST)
            assert (s["node"] == o["slots"]["node"]).all() and (s["start"] == o["slots"]["start"]).all()
            s2, r2 = F.local_search(t, s, makespan_phase2=int(r["makespan"]), flags=far.SWITCH_COST)
            oslots = np.zeros(len(s), O.SLOT_DT)
            oslots["node"], oslots["size_used"], oslots["start"] = s["node"], s["size_used"], s["start"]
            q = O.refine(prof, costs, t, oslots, int(r["makespan"]), flags=O.SWITCH_COST)
            for k in ("makespan", "moves", "swaps", "evals", "iterations", "reverted"):
                assert r2[k] == q["result"][k], k
            assert (s2["node"] == q["slots"]["node"]).all() and (s2["start"] == q["slots"]["start"]).all()
        tab = inputs.synthetic(base, 24, 200, 93)
        ms, slots, res = run_gpu(torch_dev, prof, costs, tab, flags=far.SWITCH_COST)
        check_against_oracle(O, prof, costs, tab, ms, slots, res, flags=far.SWITCH_COST)
    torch, dev = torch_dev
    F = far.Far("A100")
    d = torch.ones((2, 2, 8, 5), dtype=torch.int32, device=dev)
    with pytest.raises(far.FarError):
        F.concat_streams(d, flags=far.SWITCH_COST)


@pytest.mark.parametrize("n", [1023, 1024])
def test_variants_at_maximum_n(O, torch_dev, n):
    """The reading variants at the largest batch sizes (warp finish / fused kernel layouts)."""
    tab = np.minimum(inputs.synthetic("A100", n, 2, 5 + n, times="narrow"), 900)  # makespan bound < 2^29
    costs = inputs.reconfig_costs("A100")
    for flags in (far.BEST_IMPROVEMENT, far.SWITCH_COST, far.BEST_IMPROVEMENT | far.SWITCH_COST):
        ms, slots, res = run_gpu(torch_dev, "A100", costs, tab, flags=flags)
        check_against_oracle(O, "A100", costs, tab, ms, slots, res, flags=flags)


def test_async_calls_on_different_streams(O, torch_dev):
    """Successive asynchronous calls on one ctx on DIFFERENT streams (A, A, B, B, A ...) reuse the
    context's workspaces (two pipeline workspaces, counter slots, overflow masks): the context must
    order each reuse after the previous user's stream (include/far.h "Threading")."""
    torch, dev = torch_dev
    w = inputs.WORKLOADS["M5"]
    F = far.Far(w.profile, w.costs())
    tabs = [torch.from_numpy(w.table(count=3000, start=3000 * k)).to(dev) for k in range(5)]
    ref = []
    for d in tabs:  # single-stream reference results
        ms, _, _ = F.solve_many(d)
        ref.append(ms.clone())
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    outs = []
    for rep in range(3):
        order = [0, 0, 1, 1, 0] if rep == 0 else ([1, 0, 1, 0, 1] if rep == 1 else [0, 1, 1, 0, 0])
        for k, si in enumerate(order):
            outs.append((k, F.solve_many(tabs[k], stream=streams[si])[0]))
    torch.cuda.synchronize()
    F.sync()
    for k, ms in outs:
        assert torch.equal(ms, ref[k]), k
    oms, _ = O.far_many(w.profile, w.costs(), tabs[4].cpu().numpy())
    assert (ref[4].cpu().numpy() == oms).all()


def test_sync_calls_keep_the_async_error_flag(torch_dev):
    """A pending error of an asynchronous far_solve_many is neither consumed nor misreported by the
    synchronous host-memory calls; far_sync reports it afterwards (include/far.h "Errors")."""
    torch, dev = torch_dev
    tab = inputs.synthetic("A30", 5, 4, 3)
    bad = tab.copy()
    bad[1, 2, 1] = 0
    F = far.Far("A30")
    F.solve_many(torch.from_numpy(bad).to(dev))          # async: flags instance 1, not synced
    slots, r = F.schedule_batch(tab[0])                   # sync call on good input: OK
    assert r["status"] == 0
    ms, _, _ = F.solve_many_host(np.ascontiguousarray(tab))  # sync call on good input: OK
    assert (ms > 0).all()
    with pytest.raises(far.FarError) as e:                # the async error is still pending
        F.sync()
    assert e.value.status == 3
    F.sync()
    with pytest.raises(far.FarError) as e:                # a sync call reports its own error ...
        F.solve_many_host(np.ascontiguousarray(bad))
    assert e.value.status == 3
    F.sync()                                              # ... and leaves no flag behind


@pytest.mark.parametrize("profile,n", [("A100", 128), ("A100", 37), ("A30", 64), ("H100", 100)])
def test_general_prep_mixed_batches(O, torch_dev, profile, n):
    """Batches mixing monotone instances (far_prep_kernel<NC, true>, the merge form of phase 1) and
    non-monotone ones (listed by it and prepared by far_prep_kernel<NC, false>, the step-by-step
    growth of P:343-352) in one far_solve_many call: every instance, field and slot bit-exact, with
    and without the lower-bound pruning."""
    costs = inputs.reconfig_costs(profile)
    mono = inputs.synthetic(profile, n, 300, 41 + n)
    rnd = inputs.uniform_random(profile, n, 300, 43 + n)
    tab = np.ascontiguousarray(np.concatenate([mono, rnd])[np.random.default_rng(n).permutation(600)])
    for flags in (0, far.EXHAUSTIVE):
        ms, slots, res = run_gpu(torch_dev, profile, costs, tab, flags=flags)
        check_against_oracle(O, profile, costs, tab, ms, slots, res, flags=flags, full=True)
