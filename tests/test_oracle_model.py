"""Oracle L0 pins: the MIG model and trees against what PAPER.md states."""
import json
import os

import numpy as np
import pytest

from paper_2507_13601_b200 import inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "model.json")))


@pytest.mark.parametrize("profile", ["A30", "A100", "H100"])
def test_partition_counts(O, profile):
    # 5 A30 partitions, 19 A100/H100 partitions
    parts = O.partitions(profile)
    assert len(parts) == GOLD["partition_counts"][profile]
    nslices = {"A30": 4, "A100": 7, "H100": 7}[profile]
    for p in parts:
        # every partition: disjoint consecutive-slice instances
        cover = np.zeros(nslices, int)
        for start, size in p:
            span = 4 if (profile != "A30" and start == 0 and size == 3) else size  # 3-in-4 occupies S0..S3
            cover[start:start + span] += 1
        assert cover.max() <= 1
    assert len({tuple(sorted(p)) for p in parts}) == len(parts)


def test_a30_instances(O):
    # no 3-slice instance, no {S1,S2}
    inst = {i for p in O.partitions("A30") for i in p}
    for bad in GOLD["a30_invalid_instances"]["instances"]:
        assert tuple(bad) not in inst
    assert {s for _, s in inst} == {1, 2, 4}


def test_a100_named_partitions(O):
    parts = [sorted(p) for p in O.partitions("A100")]
    assert sorted(map(tuple, GOLD["a100_partition_4_2_1_valid"]["partition"])) in parts
    assert sorted(map(tuple, GOLD["a100_partition_2_4_1_invalid"]["partition"])) not in parts
    # exactly three partitions use {S0,S1,S2} (S3 disabled)
    assert sum(1 for p in parts if (0, 3) in p) == GOLD["a100_partitions_without_S3"]["count"]
    inst = {i for p in parts for i in p}
    assert {s for _, s in inst} == {1, 2, 3, 4, 7}


def test_tree_shape(O):
    for profile, nonleaf in (("A30", 3), ("A100", 6)):
        lo, hi, par = O.nodes(profile)
        parents = set(par[par >= 0].tolist())
        assert len(parents) == nonleaf
        # children partition their parent's interval
        for v in parents:
            ch = np.where(par == v)[0]
            assert sorted(zip(lo[ch], hi[ch]))[0][0] == lo[v]
            assert sum(hi[ch] - lo[ch]) == hi[v] - lo[v]
    assert GOLD["non_leaf_nodes"]["A30"] == 3


@pytest.mark.parametrize("profile", ["A30", "A100", "H100"])
def test_table2_constants(profile):
    # PAPER.md:177-185 Table 2 -> 1 ms ticks in the input module
    g = GOLD["table2_seconds"][profile]
    c = inputs.reconfig_costs(profile)
    assert list(inputs.SIZES[profile]) == g["sizes"]
    assert c[0].tolist() == [round(x * 1000) for x in g["create"]]
    assert c[1].tolist() == [round(x * 1000) for x in g["destroy"]]


def test_b200_same_as_a100(O):
    # B100/B200 have exactly the same MIG restrictions as the A100/H100
    assert O.partitions("H100") == O.partitions("A100")


def test_class_counts_footnote():
    # PAPER.md:995 footnote; SPEC.md:117-118 derived examples
    assert inputs.class_counts(10, (10, 10, 20, 30, 30)) == [1, 1, 2, 3, 3]
    assert inputs.class_counts(15, (50, 50, 0, 0, 0)) == [8, 7, 0, 0, 0]
    assert inputs.class_counts(0, (20, 20, 20, 20, 20)) == [0] * 5
    rng = np.random.default_rng(1)
    for _ in range(200):
        p = rng.multinomial(100, [0.2] * 5)
        n = int(rng.integers(0, 200))
        assert sum(inputs.class_counts(n, p)) == n


def test_generator_property1_and_determinism():
    # r <= 1 guarantees t(s+1) <= t(s) (property 1), and quantisation is monotone
    a = inputs.synthetic("A100", 32, 500, 7)
    assert (np.diff(a.astype(np.int64), axis=2) <= 0).all() and a.min() >= 1
    b = inputs.synthetic("A100", 32, 100, 7, start=200)
    assert (a[200:300] == b).all()
    c = inputs.synthetic("A30", 16, 300, 3, times="narrow")
    assert (np.diff(c.astype(np.int64), axis=2) <= 0).all()
    assert c[:, :, 0].min() >= 90_000 and c[:, :, 0].max() <= 100_000
    r = inputs.rodinia_like(50, 0)
    assert r.shape == (50, 16, 5) and (np.diff(r.astype(np.int64), axis=2) <= 0).all()
