"""GPU lower bounds (far_lower_bounds) and the evaluation statistics built on the CUDA path's
outputs (NEXT-1) against the oracle: bit-exact bounds, identical exact means."""
import numpy as np
import pytest

from paper_2507_13601_b200 import far, inputs, stats

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_dev():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch, torch.device("cuda:0")


@pytest.mark.parametrize("profile,n,gen", [("A100", 128, "wide"), ("A100", 32, "narrow"), ("A30", 17, "ties"),
                                           ("H100", 40, "uniform"), ("A100", 0, "wide")])
def test_lower_bounds_bitexact(O, torch_dev, profile, n, gen):
    torch, dev = torch_dev
    if gen == "ties":
        tab = inputs.small_ties(profile, n, 500, 3)
    elif gen == "uniform":
        tab = inputs.uniform_random(profile, n, 500, 4)
    else:
        tab = inputs.synthetic(profile, n, 500, 5, times=gen)
    F = far.Far(profile)
    w, h = F.lower_bounds(torch.from_numpy(tab).to(dev))
    torch.cuda.synchronize()
    w, h = w.cpu().numpy(), h.cpu().numpy()
    for i in range(tab.shape[0]):
        ow, oh = O.lower_bound(profile, tab[i])
        assert (w[i], h[i]) == (ow, oh), f"instance {i}"


@pytest.mark.parametrize("scaling", ["poor", "mixed", "good"])
@pytest.mark.parametrize("times", ["narrow", "wide"])
@pytest.mark.parametrize("n", [10, 20, 30])
def test_table_means_match_oracle(O, torch_dev, scaling, times, n):
    torch, dev = torch_dev
    costs = inputs.reconfig_costs("A100")
    tab = inputs.synthetic("A100", n, 150, 600 + n, scaling=scaling, times=times)
    F = far.Far("A100", costs)
    got = stats.solve_and_measure(F, torch.from_numpy(tab).to(dev))
    F.sync()
    want = O.table_stats("A100", costs, tab)
    assert got == want
