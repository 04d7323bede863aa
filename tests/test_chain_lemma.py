"""The prep kernel's H1 (far_prep.cuh) computes a task's growth chain a^1 -> nx(a^1) -> ... (P:341,
P:349; nx(c) = argmin_{c' > c} (size(c') t(c'), c')) as the set of suffix-minimum positions of
w_c = size(c) t(c) -- c is on the chain iff w_c <= w_c'' for every c'' > c -- with a^1 its lowest
element.  This checks that lemma against the literal walk, exhaustively on small value ranges (every
tie pattern) and on random wide values.  Pure mathematics: no CUDA, no oracle."""
import itertools
import random

SIZES = {3: (1, 2, 4), 5: (1, 2, 3, 4, 7)}


def chain_walk(t, sizes):
    w = [s * x for s, x in zip(sizes, t)]
    a = min(range(len(w)), key=lambda c: (w[c], c))  # P:341, ties -> smallest size
    chain = [a]
    while chain[-1] != len(w) - 1:  # grow to the cheapest larger size, ties -> smallest
        c = chain[-1]
        chain.append(min(range(c + 1, len(w)), key=lambda d: (w[d], d)))
    return chain


def chain_suffix_minima(t, sizes):
    w = [s * x for s, x in zip(sizes, t)]
    return [c for c in range(len(w)) if all(w[c] <= w[d] for d in range(c + 1, len(w)))]


def test_lemma_exhaustive_small():
    for nc, sizes in SIZES.items():
        for t in itertools.product(range(1, 8), repeat=nc):
            assert chain_walk(t, sizes) == chain_suffix_minima(t, sizes), t


def test_lemma_random_wide():
    rng = random.Random(7)
    for _ in range(20000):
        nc = rng.choice((3, 5))
        t = [rng.randint(1, 1 << 22) for _ in range(nc)]
        if rng.random() < 0.3:  # force ties of the products
            c, d = rng.sample(range(nc), 2)
            t[d] = t[c] * SIZES[nc][c] // SIZES[nc][d] or 1
        assert chain_walk(t, SIZES[nc]) == chain_suffix_minima(t, SIZES[nc]), t
