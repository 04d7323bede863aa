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
             "NO_REFINE")


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
