"""Seeded synthetic inputs for FAR — the ONLY module shared by the oracle side
(tests, bench cpu_baseline) and the CUDA side.

It holds none of FAR's arithmetic: it only draws per-task runtime tables
``times[I][n][|C_G|]`` (int32 ticks, 1 tick = 1 ms) shaped like the paper's
workloads, plus the Table 2 reconfiguration costs as plain data.

Generators
----------
* :func:`synthetic` — the §6.3 generator: class counts by
  the footnote rule, memory-bound share p_sup,
  t(1) ~ U(t_min, t_max), t(s+1) = (s+r)/(s+1)·t(s) with r drawn
  from the clipped normals of PAPER.md:1000-1006, transition memory→compute
  with probability 0.3 per slice step.  Readings (DESIGN.md
  §"Input recipe"): clipping = clamp; count ties → smaller size; a transitioned
  task is sub-linear from then on (literally); times are quantised to ticks with
  max(1, floor(1000·t + 0.5)) — monotone, so property 1 survives.
* :func:`rodinia_like` — config M2: the 16 frozen archetype profiles of
  ``data/rodinia_like.json`` with a per-instance input-size multiplier
  U(0.5, 2).  Rodinia-INSPIRED, not Rodinia data.
* :func:`uniform_random` — unstructured (possibly NON-monotone) times for
  edge-case parity tests (the north star: runtimes "need not be monotone").

Every generator is counter-based at chunk granularity: instance ``i`` is drawn
by ``np.random.default_rng(SeedSequence([seed, tag, i // CHUNK]))`` so any row
range can be regenerated without the rest of the table.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

import numpy as np

CHUNK = 4096

# C_A30 = {1,2,4}, C_A100 = C_H100 = {1,2,3,4,7}
SIZES = {"A30": (1, 2, 4), "A100": (1, 2, 3, 4, 7), "H100": (1, 2, 3, 4, 7)}
SLICES = {"A30": 4, "A100": 7, "H100": 7}
PROFILE_ID = {"A30": 0, "A100": 1, "H100": 2}

# PAPER.md:177-185, Table 2 (seconds) -> ticks of 1 ms.  {create: [...], destroy: [...]}
# in the profile's size order.
TABLE2_MS = {
    "A30": ([110, 120, 130], [100, 100, 100]),
    "A100": ([160, 170, 200, 210, 240], [200, 200, 210, 210, 220]),
    "H100": ([160, 210, 330, 380, 420], [210, 230, 250, 260, 260]),
}

# PAPER.md:1040-1048 presets (percent per size in C_G order)
SCALING = {
    "A100": {
        "poor": (50, 50, 0, 0, 0),
        "mixed": (20, 20, 20, 20, 20),
        "good": (0, 0, 0, 50, 50),
    },
    # A30 split used by SURVEY.md §8(d) M1/M4
    "A30": {"mixed": (34, 33, 33), "poor": (50, 50, 0), "good": (0, 50, 50)},
}
SCALING["H100"] = SCALING["A100"]
TIMES = {"wide": (1.0, 100.0), "narrow": (90.0, 100.0)}


def reconfig_costs(profile: str, zero: bool = False) -> np.ndarray:
    """int32[2][|C|] = {create[], destroy[]} in ticks (Table 2, 1 ms ticks)."""
    c, d = TABLE2_MS[profile]
    arr = np.array([c, d], dtype=np.int32)
    if zero:
        arr[:] = 0
    return arr


def class_counts(n: int, p) -> list[int]:
    """Footnote of PAPER.md:995: floor n·p_s, then +1 to argmax (n·p_s − n_s)
    while Σ < n; ties -> smaller size.  Exact integer arithmetic (percent)."""
    p = list(p)
    cnt = [(n * ps) // 100 for ps in p]
    while sum(cnt) < n:
        # deficit in units of 1/100 task
        best, bi = None, 0
        for j, ps in enumerate(p):
            d = n * ps - 100 * cnt[j]
            if best is None or d > best:
                best, bi = d, j
        cnt[bi] += 1
    return cnt


def _rng(seed: int, tag: int, chunk: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([seed, tag, chunk]))


def _synthetic_chunk(rng, B, n, sizes, nslices, p, p_sup, tmin, tmax):
    cnt = class_counts(n, p)
    cls_base = np.concatenate([np.full(c, s, dtype=np.int64) for c, s in zip(cnt, sizes)]) if n else np.zeros(0, np.int64)
    mem_base = np.zeros(n, dtype=bool)
    off = 0
    for c, s in zip(cnt, sizes):
        if s > 1:
            nm = -((-p_sup * c) // 100)  # ceil(p_sup·n_s/100)
            mem_base[off:off + nm] = True
        off += c
    perm = np.argsort(rng.random((B, n)), axis=1, kind="stable")
    cls = cls_base[perm]
    mem = mem_base[perm]
    t = rng.uniform(tmin, tmax, (B, n))
    out = np.empty((B, n, len(sizes)), dtype=np.float64)
    col = {s: j for j, s in enumerate(sizes)}
    if 1 in col:
        out[:, :, col[1]] = t
    transitioned = np.zeros((B, n), dtype=bool)
    for s in range(1, nslices):
        z = rng.standard_normal((B, n))
        u = rng.random((B, n))
        sub = s >= cls
        # memory-bound: super-linear on 1->2; on each later step it stays super-linear w.p. 0.7,
        # else it "becomes compute-bound" and moves to SUB-linear speedup for good (PAPER.md:991:
        # "moving to sub-linear speedup with a probability of 1-(1-0.3)^2 (becomes compute-bound)")
        if s > 1:
            transitioned |= mem & ~sub & (u < 0.3)
        sub = sub | transitioned
        sup = mem & ~sub
        near = ~sub & ~sup
        r = np.where(sup, np.clip(-0.25 + 0.25 * z, -0.5, 0.0),
                     np.where(near, np.clip(0.1 + 0.1 * z, 0.0, 0.2),
                              np.clip(0.75 + 0.25 * z, 0.5, 1.0)))
        t = (s + r) / (s + 1) * t
        if (s + 1) in col:
            out[:, :, col[s + 1]] = t
    ticks = np.floor(out * 1000.0 + 0.5)
    return np.maximum(ticks, 1).astype(np.int32)


def synthetic(profile: str, n: int, count: int, seed: int, scaling="mixed", times="wide",
              p_sup: int = 50, start: int = 0) -> np.ndarray:
    """§6.3 generator: int32[count][n][|C|] ticks for instances [start, start+count)."""
    sizes = SIZES[profile]
    p = SCALING[profile][scaling] if isinstance(scaling, str) else tuple(scaling)
    tmin, tmax = TIMES[times] if isinstance(times, str) else times
    return _chunked(lambda rng, B: _synthetic_chunk(rng, B, n, sizes, SLICES[profile], p, p_sup, tmin, tmax),
                    n, len(sizes), count, seed, 1, start)


def _chunked(fn, n, nc, count, seed, tag, start):
    out = np.empty((count, n, nc), dtype=np.int32)
    if count == 0:
        return out
    c0, c1 = start // CHUNK, (start + count - 1) // CHUNK
    for c in range(c0, c1 + 1):
        blk = fn(_rng(seed, tag, c), CHUNK)
        lo = max(start, c * CHUNK)
        hi = min(start + count, (c + 1) * CHUNK)
        out[lo - start:hi - start] = blk[lo - c * CHUNK:hi - c * CHUNK]
    return out


def synthetic_parallel(profile, n, count, seed, workers=None, start=0, **kw) -> np.ndarray:
    """Same table as :func:`synthetic`, generated chunk-parallel in a process pool."""
    import concurrent.futures as cf
    workers = workers or min(32, os.cpu_count() or 1)
    if count <= 4 * CHUNK or workers <= 1:
        return synthetic(profile, n, count, seed, start=start, **kw)
    sizes = SIZES[profile]
    out = np.empty((count, n, len(sizes)), dtype=np.int32)
    step = CHUNK * max(1, (count // CHUNK) // (workers * 4) or 1)
    starts = list(range(0, count, step))
    with cf.ProcessPoolExecutor(workers) as ex:
        futs = {ex.submit(synthetic, profile, n, min(step, count - s), seed, start=start + s, **kw): s
                for s in starts}
        for f in cf.as_completed(futs):
            s = futs[f]
            blk = f.result()
            out[s:s + blk.shape[0]] = blk
    return out


_DATA = os.path.join(os.path.dirname(__file__), "data", "rodinia_like.json")


def rodinia_like(count: int, seed: int, start: int = 0) -> np.ndarray:
    """Config M2: A100, n=16 (one task per archetype), int32[count][16][5] ticks."""
    with open(_DATA) as f:
        d = json.load(f)
    t1 = np.array([q["t1_s"] for q in d["profiles"]])
    sp = np.array([q["speedup"] for q in d["profiles"]])
    base = t1[:, None] / sp  # seconds at sizes (1,2,3,4,7)

    def fn(rng, B):
        mult = rng.uniform(0.5, 2.0, (B, base.shape[0]))
        t = mult[:, :, None] * base[None]
        return np.maximum(np.floor(t * 1000.0 + 0.5), 1).astype(np.int32)

    return _chunked(fn, base.shape[0], base.shape[1], count, seed, 2, start)


def uniform_random(profile: str, n: int, count: int, seed: int, lo: int = 1, hi: int = 1000,
                   start: int = 0) -> np.ndarray:
    """Unstructured times U{lo..hi} per (task, size): NOT monotone in general."""
    nc = len(SIZES[profile])
    return _chunked(lambda rng, B: rng.integers(lo, hi + 1, (B, n, nc), dtype=np.int64).astype(np.int32),
                    n, nc, count, seed, 3, start)


def small_ties(profile: str, n: int, count: int, seed: int, start: int = 0) -> np.ndarray:
    """Times in {1..4}: dense ties everywhere, to stress every tie-break rule."""
    return uniform_random(profile, n, count, seed, 1, 4, start)


def monotone_ties(profile: str, n: int, count: int, seed: int, hi: int = 6, start: int = 0) -> np.ndarray:
    """Monotone (property 1) times in {1..hi}, non-increasing in the size: equal times along a
    task's sizes and across tasks everywhere (stresses the growth tie rules)."""
    nc = len(SIZES[profile])
    return _chunked(lambda rng, B: -np.sort(-rng.integers(1, hi + 1, (B, n, nc)), axis=2).astype(np.int32),
                    n, nc, count, seed, 4, start)


@dataclass(frozen=True)
class Workload:
    """A BASELINE.json config as a concrete seeded recipe."""
    name: str
    profile: str
    n: int
    count: int
    seed: int
    kind: str = "synthetic"      # synthetic | rodinia
    scaling: str = "mixed"
    times: str = "wide"
    zero_reconfig: bool = False

    def table(self, count=None, start=0, parallel=False) -> np.ndarray:
        c = self.count if count is None else count
        if self.kind == "rodinia":
            return rodinia_like(c, self.seed, start)
        if parallel:
            return synthetic_parallel(self.profile, self.n, c, self.seed, scaling=self.scaling, times=self.times,
                                      start=start)
        return synthetic(self.profile, self.n, c, self.seed, scaling=self.scaling, times=self.times, start=start)

    def costs(self) -> np.ndarray:
        return reconfig_costs(self.profile, self.zero_reconfig)


WORKLOADS = {
    "M1": Workload("M1_A30_n8_zero_reconfig", "A30", 8, 10_000, 0, zero_reconfig=True),
    "M2": Workload("M2_A100_n16_rodinia_like", "A100", 16, 10_000, 0, kind="rodinia"),
    "M3": Workload("M3_A100_n32_100k", "A100", 32, 100_000, 3),
    "M4_A30": Workload("M4_A30_stream_64x64", "A30", 64, 64, 4),
    "M4_A100": Workload("M4_A100_stream_64x64", "A100", 64, 64, 4),
    "M5": Workload("M5_A100_n128_1M", "A100", 128, 1_000_000, 5),
}
