"""GPU schedule export and checking (include/far.h far_schedule_events / far_validate_schedules,
SURVEY.md §8(f) NEXT-4) against the oracle: the reconfiguration events of every FAR output equal
the oracle's event list, and the violation counts of valid and corrupted schedules equal
orc_validate's, element by element."""
import numpy as np
import pytest

from oracle import oracle as O_mod
from paper_2507_13601_b200 import far, inputs

pytestmark = pytest.mark.gpu

OEV_DT = np.dtype([("kind", "<i4"), ("node", "<i4"), ("start", "<i8"), ("dur", "<i8")])


@pytest.fixture(scope="module")
def torch_dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch, torch.device("cuda:0")


def to_oracle_slots(s):
    o = np.zeros(len(s), O_mod.SLOT_DT)
    o["node"], o["size_used"], o["start"] = s["node"], s["size_used"], s["start"]
    return o


def to_oracle_events(e):
    o = np.zeros(len(e), OEV_DT)
    for k in ("kind", "node", "start", "dur"):
        o[k] = e[k]
    return o


def ordered(ev):
    """events as tuples in (start, node, kind) order (zero-duration events may share a start)."""
    return sorted((int(e["start"]), int(e["node"]), int(e["kind"]), int(e["dur"])) for e in ev)


def solve_and_events(torch_dev, profile, costs, tab, flags=0):
    torch, dev = torch_dev
    F = far.Far(profile, costs)
    d = torch.from_numpy(np.ascontiguousarray(tab)).to(dev)
    ms, sd, rs = F.solve_many(d, flags=flags)
    ev, nev, ems = F.schedule_events(d, sd, flags=flags & far.ZERO_RECONFIG)
    viol = F.validate_schedules(d, sd, ev, nev, flags=flags & far.ZERO_RECONFIG)
    torch.cuda.synchronize()
    F.sync()
    return F, d, sd, ms.cpu().numpy(), far.slots_np(sd), far.events_np(ev, nev), nev.cpu().numpy(), \
        ems.cpu().numpy(), viol.cpu().numpy()


CASES = [("M1", None, 300), ("M2", None, 300), ("M3", None, 200), ("M5", None, 60),
         ("A30", "ties", 200), ("A100", "ties", 200), ("A100", "monoties", 200), ("H100", "uniform", 100)]


def case_table(wname, gen, count):
    if gen is None:
        w = inputs.WORKLOADS[wname]
        return w.profile, w.costs(), w.table(count=count), 0
    profile = wname
    costs = inputs.reconfig_costs(profile)
    if gen == "ties":
        return profile, costs, inputs.small_ties(profile, 20, count, 11), 0
    if gen == "monoties":
        return profile, costs, inputs.monotone_ties(profile, 24, count, 12), 0
    return profile, costs, inputs.uniform_random(profile, 16, count, 13), 0


@pytest.mark.parametrize("wname,gen,count", CASES)
@pytest.mark.parametrize("flags", [0, far.NO_REFINE, far.NO_GUARD])
def test_events_match_oracle(O, torch_dev, wname, gen, count, flags):
    profile, costs, tab, _ = case_table(wname, gen, count)
    F, d, sd, ms, slots, evs, nev, ems, viol = solve_and_events(torch_dev, profile, costs, tab, flags=flags)
    assert (ems == ms).all(), "the replay of a FAR output reproduces its makespan (fixpoint)"
    assert (viol == 0).all(), f"infeasible outputs at {np.nonzero(viol)[0][:10]}"
    for i in range(tab.shape[0]):
        o = O.far(profile, costs, tab[i], flags=flags & (O.NO_REFINE | O.NO_GUARD | O.ZERO_RECONFIG))
        assert ordered(evs[i]) == ordered(o["events"]), f"events differ, instance {i}"
        assert O.validate(profile, costs, tab[i], to_oracle_slots(slots[i]), to_oracle_events(evs[i])) == 0


def test_zero_reconfig_and_empty(O, torch_dev):
    profile = "A100"
    costs = inputs.reconfig_costs(profile, zero=True)
    tab = inputs.synthetic(profile, 12, 100, 21)
    F, d, sd, ms, slots, evs, nev, ems, viol = solve_and_events(torch_dev, profile, costs, tab)
    assert (viol == 0).all() and (ems == ms).all()
    for i in range(tab.shape[0]):
        o = O.far(profile, costs, tab[i])
        assert ordered(evs[i]) == ordered(o["events"])
    torch, dev = torch_dev
    e = torch.zeros((3, 0, 5), dtype=torch.int32, device=dev)
    s = torch.zeros((3, 0, 8), dtype=torch.uint8, device=dev)
    ev, nev, ems = F.schedule_events(e, s)
    torch.cuda.synchronize()
    assert (nev.cpu().numpy() == 0).all() and (ems.cpu().numpy() == 0).all()


def perturb(rng, profile, slots, evs, tab, nlo, nhi):
    """Random corruptions of a schedule and its events (start shifts, node/size changes,
    event shifts / durations / nodes, dropped and duplicated events)."""
    s = slots.copy()
    e = evs.copy()
    kind = rng.integers(0, 7)
    n = len(s)
    if kind == 0 and n:
        j = rng.integers(n)
        s["start"][j] = max(0, int(s["start"][j]) + int(rng.integers(-50, 50)))
    elif kind == 1 and n:
        j = rng.integers(n)
        s["node"][j] = rng.integers(len(nlo))
        s["size_used"][j] = nhi[s["node"][j]] - nlo[s["node"][j]]
    elif kind == 2 and n:
        j = rng.integers(n)
        s["start"][j] = -1 if rng.random() < 0.3 else int(s["start"][j]) + 1
    elif kind == 3 and len(e):
        g = rng.integers(len(e))
        e["start"][g] += int(rng.integers(-20, 20))
    elif kind == 4 and len(e):
        g = rng.integers(len(e))
        e["dur"][g] += 1
    elif kind == 5 and len(e):
        e = np.delete(e, rng.integers(len(e)))
    elif kind == 6 and len(e):
        e = np.concatenate([e, e[rng.integers(len(e)):][:1]])
    return s, e


@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_validator_counts_match_oracle(O, torch_dev, profile):
    torch, dev = torch_dev
    costs = inputs.reconfig_costs(profile)
    tab = inputs.synthetic(profile, 14, 400, 31)
    F, d, sd, ms, slots, evs, nev, ems, viol = solve_and_events(torch_dev, profile, costs, tab)
    lo, hi, _ = F.node_table()
    rng = np.random.default_rng(5)
    cap = 2 * F.nnodes
    S = np.zeros((tab.shape[0], tab.shape[1]), far.SLOT_DT)
    E = np.zeros((tab.shape[0], cap), far.EVENT_DT)
    NE = np.zeros(tab.shape[0], np.int32)
    for i in range(tab.shape[0]):
        s, e = slots[i], evs[i]
        for _ in range(rng.integers(1, 3)):
            s, e = perturb(rng, profile, s, e, tab[i], lo, hi)
        e = e[:cap]
        S[i], E[i, :len(e)], NE[i] = s, e, len(e)
    dS = torch.from_numpy(S.view(np.uint8).reshape(tab.shape[0], tab.shape[1], 8)).to(dev)
    dE = torch.from_numpy(E.view(np.uint8).reshape(tab.shape[0], cap, 16)).to(dev)
    dN = torch.from_numpy(NE).to(dev)
    v = F.validate_schedules(d, dS, dE, dN).cpu().numpy()
    want = np.array([O.validate(profile, costs, tab[i], to_oracle_slots(S[i]), to_oracle_events(E[i, :NE[i]]))
                     for i in range(tab.shape[0])])
    assert (v == want).all(), f"mismatch at {np.nonzero(v != want)[0][:10]}: gpu {v[v != want][:5]} oracle {want[v != want][:5]}"
    assert (want > 0).mean() > 0.5  # the corruptions are mostly detected


def test_full_size_m5_feasible(torch_dev):
    """Every one of the 1M M5 outputs is feasible (constraints 1-3 + lifecycles) and its event
    replay reproduces its makespan -- a property check at full size, no oracle involved."""
    torch, dev = torch_dev
    w = inputs.WORKLOADS["M5"]
    host = inputs.synthetic_parallel(w.profile, w.n, w.count, w.seed, scaling=w.scaling, times=w.times)
    F = far.Far(w.profile, w.costs())
    d = torch.from_numpy(host).to(dev)
    ms, sd, rs = F.solve_many(d)
    ev, nev, ems = F.schedule_events(d, sd)
    viol = F.validate_schedules(d, sd, ev, nev)
    torch.cuda.synchronize()
    F.sync()
    assert int((viol != 0).sum().item()) == 0
    assert bool((ems == ms).all().item())
    assert int((nev <= 0).sum().item()) == 0
