"""GPU parity of the §4 multi-batch fold (far_concat_streams) against the oracle."""
import numpy as np
import pytest

from paper_2507_13601_b200 import far, inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch, torch.device("cuda:0")


def run_streams(torch_dev, profile, costs, tab, **kw):
    torch, dev = torch_dev
    F = far.Far(profile, costs)
    sm, off, sd, br, se = F.concat_streams(torch.from_numpy(np.ascontiguousarray(tab)).to(dev), **kw)
    torch.cuda.synchronize()
    F.sync()
    return (sm.cpu().numpy(), off.cpu().numpy(), far.slots_np(sd), far.results_np(br), se.cpu().numpy())


def check(O, profile, costs, tab, out, **kw):
    sm, off, slots, res, seam = out
    for s in range(tab.shape[0]):
        o = O.stream(profile, costs, tab[s], **kw)
        assert o["violations"] == 0
        assert sm[s, 0] == o["makespan"] and sm[s, 1] == o["trivial"], f"stream {s} makespans"
        assert (off[s] == o["offsets"]).all(), f"stream {s} offsets {np.nonzero(off[s] != o['offsets'])[0][:5]}"
        assert (seam[s] == o["seam"]).all(), f"stream {s} seam info"
        assert (slots[s]["node"] == o["slots"]["node"]).all(), f"stream {s} nodes"
        assert (slots[s]["start"] == o["slots"]["start"]).all(), f"stream {s} starts"
        for k in ("makespan", "alloc_index", "moves", "swaps", "evals"):
            assert (res[s][k] == o["results"][k]).all(), f"stream {s} {k}"


@pytest.mark.parametrize("wname", ["M4_A30", "M4_A100"])
def test_m4_stream_bitexact(O, torch_dev, wname):
    w = inputs.WORKLOADS[wname]
    tab = w.table(count=64)[None]          # one stream of 64 batches x 64 tasks
    out = run_streams(torch_dev, w.profile, w.costs(), tab)
    check(O, w.profile, w.costs(), tab, out)


@pytest.mark.parametrize("profile", ["A30", "A100", "H100"])
@pytest.mark.parametrize("n", [1, 5, 10, 30])
def test_many_streams(O, torch_dev, profile, n):
    tab = inputs.synthetic(profile, n, 12 * 9, 40 + n).reshape(12, 9, n, -1)
    for costs in (inputs.reconfig_costs(profile), inputs.reconfig_costs(profile, zero=True)):
        out = run_streams(torch_dev, profile, costs, tab)
        check(O, profile, costs, tab, out)


@pytest.mark.parametrize("gen", ["ties", "uniform", "narrow"])
def test_stream_edge_inputs(O, torch_dev, gen):
    profile = "A100"
    n = 12
    if gen == "ties":
        t = inputs.small_ties(profile, n, 64, 3)
    elif gen == "uniform":
        t = inputs.uniform_random(profile, n, 64, 4)
    else:
        t = inputs.synthetic(profile, n, 64, 5, times="narrow")
    tab = t.reshape(8, 8, n, -1)
    costs = inputs.reconfig_costs(profile)
    out = run_streams(torch_dev, profile, costs, tab)
    check(O, profile, costs, tab, out)
    out = run_streams(torch_dev, profile, costs, tab, max_iterations=2)
    check(O, profile, costs, tab, out, max_iterations=2)


@pytest.mark.parametrize("profile", ["A30", "A100"])
def test_no_seam_moves_flag(O, torch_dev, profile):
    # FAR_NO_SEAM_MOVES (reversal + seam offset only; Table 7's p_rev) against the oracle
    tab = inputs.synthetic(profile, 10, 8 * 6, 77).reshape(8, 6, 10, -1)
    costs = inputs.reconfig_costs(profile)
    out = run_streams(torch_dev, profile, costs, tab, flags=far.NO_SEAM_MOVES)
    check(O, profile, costs, tab, out, flags=O.NO_SEAM_MOVES)
    assert (out[4][:, :, 1:3] == 0).all()


@pytest.mark.parametrize("scaling,times", [("poor", "narrow"), ("mixed", "wide"), ("good", "narrow")])
def test_concat_and_multibatch_statistics(O, torch_dev, scaling, times):
    # Tables 7-9 statistics from the CUDA path equal the oracle's exact means
    from paper_2507_13601_b200 import stats
    torch, dev = torch_dev
    costs = inputs.reconfig_costs("A100")
    F = far.Far("A100", costs)
    two = inputs.synthetic("A100", 10, 2 * 60, 300, scaling=scaling, times=times).reshape(60, 2, 10, -1)
    got = stats.concat_means(F, torch.from_numpy(two).to(dev))
    assert got == O.concat_stats("A100", costs, two)
    long = inputs.synthetic("A100", 12, 101, 301, scaling=scaling, times=times)
    assert stats.multi_batch_p(F, torch.from_numpy(long).to(dev)) == O.multi_batch_p("A100", costs, long)
    F.sync()


def test_grow_ties_streams(O, torch_dev):
    tab = inputs.small_ties("A100", 12, 6 * 5, 78).reshape(6, 5, 12, -1)
    costs = inputs.reconfig_costs("A100")
    out = run_streams(torch_dev, "A100", costs, tab, flags=far.GROW_TIES)
    check(O, "A100", costs, tab, out, flags=O.GROW_TIES)


def test_best_improvement_streams(O, torch_dev):
    tab = inputs.synthetic("A30", 16, 4 * 6, 79).reshape(4, 6, 16, -1)
    costs = inputs.reconfig_costs("A30")
    out = run_streams(torch_dev, "A30", costs, tab, flags=far.BEST_IMPROVEMENT)
    check(O, "A30", costs, tab, out, flags=O.BEST_IMPROVEMENT)


def _oracle_stream(args):
    from oracle import oracle as O
    profile, costs, t = args
    o = O.stream(profile, costs, t)
    return (o["makespan"], o["trivial"], o["offsets"], o["seam"], o["violations"],
            o["results"]["makespan"], o["results"]["moves"], o["results"]["swaps"], o["results"]["evals"],
            o["slots"]["node"], o["slots"]["start"])


@pytest.mark.parametrize("wname", ["M4_A30", "M4_A100"])
def test_m4_full_size_bitexact(O, torch_dev, wname):
    """BASELINE configs[3] at the bench's size: all 1024 streams x 64 batches x 64 tasks, every
    stream makespan, offset, seam record, per-batch report and task slot bit-exact (oracle over the
    host cores)."""
    import concurrent.futures as cf
    import os
    w = inputs.WORKLOADS[wname]
    S = 1024
    tab = inputs.synthetic_parallel(w.profile, w.n, S * 64, w.seed).reshape(S, 64, w.n, -1)
    sm, off, slots, res, seam = run_streams(torch_dev, w.profile, w.costs(), tab)
    with cf.ProcessPoolExecutor(os.cpu_count() or 1) as ex:
        outs = list(ex.map(_oracle_stream, [(w.profile, w.costs(), tab[s]) for s in range(S)], chunksize=16))
    for s, o in enumerate(outs):
        assert o[4] == 0
        assert sm[s, 0] == o[0] and sm[s, 1] == o[1], f"stream {s} makespans"
        assert (off[s] == o[2]).all() and (seam[s] == o[3]).all(), f"stream {s} offsets / seams"
        assert (res[s]["makespan"] == o[5]).all() and (res[s]["moves"] == o[6]).all(), f"stream {s} reports"
        assert (res[s]["swaps"] == o[7]).all() and (res[s]["evals"] == o[8]).all(), f"stream {s} reports"
        assert (slots[s]["node"] == o[9]).all() and (slots[s]["start"] == o[10]).all(), f"stream {s} slots"
