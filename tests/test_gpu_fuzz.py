"""Randomised parity sweep: many random (profile, forest size, n, batch size, input generator,
reconfiguration costs, flags, iteration cap, min-improvement) combinations, the CUDA path
against the oracle on every instance (makespans and every report field; full schedules on a
sample).  Seeded, so a failure names a reproducible case."""
import os

import numpy as np
import pytest

from paper_2507_13601_b200 import far, inputs
from test_gpu_parity import check_against_oracle, run_gpu

pytestmark = pytest.mark.gpu

FLAG_POOL = ("NO_GUARD", "NONEMPTY_ALT", "GROW_TIES", "EXHAUSTIVE", "BEST_IMPROVEMENT", "ZERO_RECONFIG",
             "NO_REFINE", "SWITCH_COST")


@pytest.fixture(scope="module")
def torch_dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch, torch.device("cuda:0")


def case(seed):
    rng = np.random.default_rng(seed)
    base = ["A30", "A100", "H100"][rng.integers(3)]
    g = int(rng.choice([1, 1, 1, 2, 3]))
    prof = base if g == 1 else f"{base}x{g}"
    n = int(rng.choice([0, 1, 2, 5, 9, 16, 31, 33, 64, 100, 128, 200, 256] + ([300, 511] if g == 1 else [])))
    count = int(rng.choice([1, 7, 40, 255, 256, 300])) if n <= 128 else int(rng.choice([1, 5, 20]))
    gen = ["mixed", "poor", "good", "narrow", "uniform", "ties", "monoties"][rng.integers(7)]
    s = int(rng.integers(1 << 30))
    if gen in ("mixed", "poor", "good", "narrow"):
        tab = inputs.synthetic(base, n, count, s, scaling="mixed" if gen == "narrow" else gen,
                               times="narrow" if gen == "narrow" else "wide")
    elif gen == "uniform":
        tab = inputs.uniform_random(base, n, count, s)
    elif gen == "ties":
        tab = inputs.small_ties(base, n, count, s)
    else:
        tab = inputs.monotone_ties(base, n, count, s)
    kind = rng.integers(3)
    if kind == 0:
        costs = inputs.reconfig_costs(base)
    elif kind == 1:
        costs = inputs.reconfig_costs(base, zero=True)
    else:
        costs = rng.integers(0, 3000, size=(2, len(inputs.SIZES[base]))).astype(np.int32)
    flags = 0
    for f in FLAG_POOL:
        if rng.random() < 0.2:
            flags |= getattr(far, f)
    max_it = int(rng.choice([0, 1, 3, 100]))
    ppm = int(rng.choice([0, 0, 0, 5000]))
    return prof, costs, np.ascontiguousarray(tab), flags, max_it, ppm


@pytest.mark.parametrize("seed", range(int(os.environ.get("FAR_FUZZ_SEEDS", "120"))))
def test_random_configs(O, torch_dev, seed):
    prof, costs, tab, flags, max_it, ppm = case(seed)
    ms, slots, res = run_gpu(torch_dev, prof, costs, tab, flags=flags, max_iterations=max_it, min_improvement_ppm=ppm)
    check_against_oracle(O, prof, costs, tab, ms, slots, res, flags=flags, max_iterations=max_it, ppm=ppm,
                         full=tab.shape[0] * max(tab.shape[1], 1) <= 4000)


def stream_case(seed):
    rng = np.random.default_rng(10_000 + seed)
    base = ["A30", "A100", "H100"][rng.integers(3)]
    S, B = int(rng.integers(1, 5)), int(rng.integers(1, 9))
    n = int(rng.choice([1, 2, 5, 12, 24, 40, 64]))
    gen = ["mixed", "narrow", "ties", "monoties"][rng.integers(4)]
    s = int(rng.integers(1 << 30))
    if gen == "ties":
        tab = inputs.small_ties(base, n, S * B, s)
    elif gen == "monoties":
        tab = inputs.monotone_ties(base, n, S * B, s)
    else:
        tab = inputs.synthetic(base, n, S * B, s, times="narrow" if gen == "narrow" else "wide")
    tab = np.ascontiguousarray(tab.reshape(S, B, n, -1))
    kind = rng.integers(3)
    costs = (inputs.reconfig_costs(base) if kind == 0 else inputs.reconfig_costs(base, zero=True) if kind == 1
             else rng.integers(0, 3000, size=(2, len(inputs.SIZES[base]))).astype(np.int32))
    flags = 0
    for f in ("NO_SEAM_MOVES", "GROW_TIES", "NONEMPTY_ALT", "BEST_IMPROVEMENT", "NO_GUARD", "ZERO_RECONFIG"):
        if rng.random() < 0.2:
            flags |= getattr(far, f)
    return base, costs, tab, flags


@pytest.mark.parametrize("seed", range(int(os.environ.get("FAR_FUZZ_STREAM_SEEDS", "40"))))
def test_random_streams(O, torch_dev, seed):
    from test_gpu_stream import check, run_streams
    base, costs, tab, flags = stream_case(seed)
    out = run_streams(torch_dev, base, costs, tab, flags=flags)
    oflags = 0
    for f in ("NO_SEAM_MOVES", "GROW_TIES", "NONEMPTY_ALT", "BEST_IMPROVEMENT", "NO_GUARD", "ZERO_RECONFIG"):
        if flags & getattr(far, f):
            oflags |= getattr(O, f)
    check(O, base, costs, tab, out, flags=oflags)


@pytest.mark.parametrize("seed", range(int(os.environ.get("FAR_FUZZ_CHECK_SEEDS", "40"))))
def test_random_events_and_validator(O, torch_dev, seed):
    """Events of random FAR outputs equal the oracle's; valid outputs have no violations, and a
    randomly corrupted copy gets the oracle's violation count."""
    from test_gpu_check import ordered, solve_and_events, to_oracle_events, to_oracle_slots
    prof, costs, tab, flags, _, _ = case(20_000 + seed)
    if "x" in prof or tab.shape[1] == 0:
        pytest.skip("events / validator: single-GPU trees, n > 0")
    tab = tab[:40]
    flags &= far.NO_REFINE | far.NO_GUARD | far.ZERO_RECONFIG | far.GROW_TIES | far.NONEMPTY_ALT
    F, d, sd, ms, slots, evs, nev, ems, viol = solve_and_events(torch_dev, prof, costs, tab, flags=flags)
    assert (ems == ms).all() and (viol == 0).all()
    oc = inputs.reconfig_costs(prof, zero=True) if flags & far.ZERO_RECONFIG else costs
    oflags = 0
    for f in ("NO_REFINE", "NO_GUARD", "ZERO_RECONFIG", "GROW_TIES", "NONEMPTY_ALT"):
        if flags & getattr(far, f):
            oflags |= getattr(O, f)
    for i in range(tab.shape[0]):
        o = O.far(prof, costs, tab[i], flags=oflags)
        assert ordered(evs[i]) == ordered(o["events"]), f"events differ, instance {i}"
        assert O.validate(prof, oc, tab[i], to_oracle_slots(slots[i]), to_oracle_events(evs[i])) == 0
    # corrupted copies: the GPU violation counts equal the oracle's
    from test_gpu_check import perturb
    torch, dev = torch_dev
    lo, hi, _ = F.node_table()
    rng = np.random.default_rng(30_000 + seed)
    cap = 2 * F.nnodes
    S = np.zeros((tab.shape[0], tab.shape[1]), far.SLOT_DT)
    E = np.zeros((tab.shape[0], cap), far.EVENT_DT)
    NE = np.zeros(tab.shape[0], np.int32)
    for i in range(tab.shape[0]):
        s_, e_ = slots[i], evs[i]
        for _ in range(rng.integers(1, 3)):
            s_, e_ = perturb(rng, prof, s_, e_, tab[i], lo, hi)
        e_ = e_[:cap]
        S[i], E[i, :len(e_)], NE[i] = s_, e_, len(e_)
    dS = torch.from_numpy(S.view(np.uint8).reshape(tab.shape[0], tab.shape[1], 8)).to(dev)
    dE = torch.from_numpy(E.view(np.uint8).reshape(tab.shape[0], cap, 16)).to(dev)
    v = F.validate_schedules(d, dS, dE, torch.from_numpy(NE).to(dev), flags=flags & far.ZERO_RECONFIG).cpu().numpy()
    want = np.array([O.validate(prof, oc, tab[i], to_oracle_slots(S[i]), to_oracle_events(E[i, :NE[i]]))
                     for i in range(tab.shape[0])])
    assert (v == want).all(), f"validator mismatch at {np.nonzero(v != want)[0][:10]}"


@pytest.mark.parametrize("seed", range(int(os.environ.get("FAR_FUZZ_LOCAL_SEEDS", "30"))))
def test_random_local_search(O, torch_dev, seed):
    """far_local_search on arbitrary schedules (random hosting node and size per task, random
    starts -- the node lists follow the start order, unsorted by duration) equals the oracle's
    refine + replay + guard."""
    rng = np.random.default_rng(40_000 + seed)
    base = ["A30", "A100", "H100"][rng.integers(3)]
    g = int(rng.choice([1, 1, 2]))
    prof = base if g == 1 else f"{base}x{g}"
    n = int(rng.integers(1, 48))
    t = inputs.synthetic(base, n, 1, int(rng.integers(1 << 30)))[0]
    costs = inputs.reconfig_costs(base) if rng.random() < 0.5 else inputs.reconfig_costs(base, zero=True)
    lo, hi, _ = O.nodes(prof)
    sizes = inputs.SIZES[base]
    s = np.zeros(n, far.SLOT_DT)
    for j in range(n):
        v = int(rng.integers(len(lo)))
        z = int(hi[v] - lo[v])
        if z == 4 and base != "A30" and rng.random() < 0.5:
            z = 3  # the A100/H100 {S0..S3} node also hosts size-3 tasks
        s["node"][j], s["size_used"][j], s["start"][j] = v, z, int(rng.integers(0, 2000))
    ms_in = int(max(s["start"][j] + t[j][sizes.index(int(s["size_used"][j]))] for j in range(n)))
    F = far.Far(prof, costs)
    oslots = np.zeros(n, O.SLOT_DT)
    oslots["node"], oslots["size_used"], oslots["start"] = s["node"], s["size_used"], s["start"]
    for fname in ("", "NO_GUARD", "NONEMPTY_ALT", "BEST_IMPROVEMENT", "SWITCH_COST"):
        flags = getattr(far, fname) if fname else 0
        oflags = getattr(O, fname) if fname else 0
        mi = int(rng.choice([0, 1, 100]))
        s2, r2 = F.local_search(t, s, makespan_phase2=ms_in, flags=flags, max_iterations=mi)
        q = O.refine(prof, costs, t, oslots, ms_in, flags=oflags, max_iterations=mi)
        for k in ("makespan", "moves", "swaps", "evals", "iterations", "reverted"):
            assert r2[k] == q["result"][k], (fname, k)
        assert (s2["node"] == q["slots"]["node"]).all() and (s2["start"] == q["slots"]["start"]).all(), fname
