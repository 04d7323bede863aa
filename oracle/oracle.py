"""ctypes wrapper of liboracle.so — the CPU ORACLE of FAR.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  It never touches
the CUDA path (paper_2507_13601_b200/) and the CUDA path never touches it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SOURCES = ["far_oracle.cpp"]

PROFILES = {"A30": 0, "A100": 1, "H100": 2}
NO_REFINE, NO_GUARD, ZERO_RECONFIG, NONEMPTY_ALT, NO_SEAM_MOVES, GROW_TIES, BEST_IMPROVEMENT, SWITCH_COST = \
    1, 2, 4, 32, 64, 128, 256, 512


def build(force: bool = False) -> str:
    srcs = [os.path.join(HERE, s) for s in SOURCES if os.path.exists(os.path.join(HERE, s))]
    if force or not os.path.exists(LIB) or any(os.path.getmtime(s) > os.path.getmtime(LIB) for s in srcs
                                               + [os.path.join(HERE, "far_oracle.h")]):
        subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-Wall", "-o", LIB] + srcs)
    return LIB


class Slot(C.Structure):
    _fields_ = [("node", C.c_int32), ("size_used", C.c_int32), ("start", C.c_int64)]


class Event(C.Structure):
    _fields_ = [("kind", C.c_int32), ("node", C.c_int32), ("start", C.c_int64), ("dur", C.c_int64)]


class Result(C.Structure):
    _fields_ = [("makespan", C.c_int64), ("makespan_phase2", C.c_int64), ("evals", C.c_int64),
                ("events", C.c_int64), ("alloc_index", C.c_int32), ("family_size", C.c_int32),
                ("moves", C.c_int32), ("swaps", C.c_int32), ("reverted", C.c_int32),
                ("iterations", C.c_int32)]

    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


SLOT_DT = np.dtype([("node", "<i4"), ("size_used", "<i4"), ("start", "<i8")])
RESULT_DT = np.dtype([("makespan", "<i8"), ("makespan_phase2", "<i8"), ("evals", "<i8"), ("events", "<i8"),
                      ("alloc_index", "<i4"), ("family_size", "<i4"), ("moves", "<i4"), ("swaps", "<i4"),
                      ("reverted", "<i4"), ("iterations", "<i4")])
MAX_EVENTS = 256  # >= 2 events per node of the largest forest (8 x 13 nodes)


class OracleError(RuntimeError):
    pass


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        p = C.c_void_p
        for name, args, res in [
            ("orc_num_sizes", [C.c_int], C.c_int),
            ("orc_num_nodes", [C.c_int], C.c_int),
            ("orc_num_slices", [C.c_int], C.c_int),
            ("orc_nodes", [C.c_int, p, p, p], C.c_int),
            ("orc_partitions", [C.c_int, p, p, C.c_int, C.c_int], C.c_int),
            ("orc_family", [C.c_int, p, C.c_int, p, C.c_int], C.c_int),
            ("orc_schedule_allocation", [C.c_int, p, p, C.c_int, p, p, p, p, p, p], C.c_int),
            ("orc_far", [C.c_int, p, p, C.c_int, C.c_int32, C.c_int32, C.c_uint32, p, p, p, p], C.c_int),
            ("orc_refine", [C.c_int, p, p, C.c_int, C.c_int32, C.c_int32, C.c_uint32, p, p, p, p], C.c_int),
            ("orc_bruteforce", [C.c_int, p, C.c_int], C.c_int64),
            ("orc_validate", [C.c_int, p, p, C.c_int, p, p, C.c_int32], C.c_int),
            ("orc_validate_flags", [C.c_int, p, p, C.c_int, p, p, C.c_int32, C.c_uint32], C.c_int),
            ("orc_schedule_allocation_flags", [C.c_int, p, p, C.c_int, p, C.c_uint32, p, p, p, p, p], C.c_int),
            ("orc_lower_bound", [C.c_int, p, C.c_int, p, p], C.c_int),
            ("orc_far_many", [C.c_int, p, p, C.c_int64, C.c_int, C.c_int32, C.c_int32, C.c_uint32, p, p], C.c_int),
            ("orc_far_many_slots", [C.c_int, p, p, C.c_int64, C.c_int, C.c_int32, C.c_int32, C.c_uint32, p, p, p],
             C.c_int),
            ("orc_seam_offset_simple", [C.c_int, p, p], C.c_int64),
        ]:
            f = getattr(_lib, name)
            f.argtypes, f.restype = args, res
        if hasattr(_lib, "orc_stream"):
            _lib.orc_stream.argtypes = [C.c_int, p, p, C.c_int, C.c_int, C.c_int32, C.c_int32, C.c_uint32,
                                        p, p, p, p, p, p]
            _lib.orc_stream.restype = C.c_int
            _lib.orc_stream_ends.argtypes = [C.c_int, p, p, C.c_int, C.c_int, C.c_int32, C.c_int32, C.c_uint32,
                                             p, p, p, p, p, p, p]
            _lib.orc_stream_ends.restype = C.c_int
            _lib.orc_stream_probe.argtypes = [C.c_int, p, p, C.c_int, C.c_int, C.c_int, C.c_int64, p, p]
            _lib.orc_stream_probe.restype = C.c_int
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _times(times):
    return np.ascontiguousarray(times, dtype=np.int32)


def _costs(costs):
    return None if costs is None else np.ascontiguousarray(costs, dtype=np.int32)


def _check(rc):
    if rc != 0:
        raise OracleError(f"oracle error {rc}")


def pid(profile):
    """'A30' / 'A100' / 'H100', or 'A30x2' ... 'A100x8' for multi-target FAR (g trees)."""
    if isinstance(profile, str):
        base, _, g = profile.partition("x")
        return PROFILES[base] | (int(g) << 8 if g else 0)
    return int(profile)


def nodes(profile):
    N = lib().orc_num_nodes(pid(profile))
    lo, hi, par = (np.zeros(N, np.int32) for _ in range(3))
    lib().orc_nodes(pid(profile), _ptr(lo), _ptr(hi), _ptr(par))
    return lo, hi, par


def partitions(profile):
    maxp, maxi = 64, 8
    out = np.zeros((maxp, maxi, 2), np.int32)
    cnt = np.zeros(maxp, np.int32)
    k = lib().orc_partitions(pid(profile), _ptr(out), _ptr(cnt), maxp, maxi)
    return [[tuple(map(int, out[j, q])) for q in range(cnt[j])] for j in range(k)]


def family(profile, times, flags=0):
    t = _times(times)
    n = t.shape[0]
    nc = lib().orc_num_sizes(pid(profile))
    maxK = 1 + n * (nc - 1) + 1
    out = np.zeros((maxK, n), np.int32)
    K = lib().orc_family_flags(pid(profile), _ptr(t), n, C.c_uint32(flags), _ptr(out), maxK)
    if K < 0:
        raise OracleError(K)
    return out[:K].copy()


def schedule_allocation(profile, costs, times, alloc, flags=0):
    t = _times(times)
    n = t.shape[0]
    a = np.ascontiguousarray(alloc, dtype=np.int32)
    slots = np.zeros(n, SLOT_DT)
    ev = np.zeros(MAX_EVENTS, dtype=[("kind", "<i4"), ("node", "<i4"), ("start", "<i8"), ("dur", "<i8")])
    nev = np.zeros(1, np.int32)
    ms = np.zeros(1, np.int64)
    pops = np.zeros(1, np.int64)
    _check(lib().orc_schedule_allocation_flags(pid(profile), _ptr(_costs(costs)), _ptr(t), n, _ptr(a), flags,
                                               _ptr(slots), _ptr(ev), _ptr(nev), _ptr(ms), _ptr(pops)))
    return {"slots": slots, "events": ev[:nev[0]].copy(), "makespan": int(ms[0]), "pops": int(pops[0])}


def far(profile, costs, times, max_iterations=100, min_improvement_ppm=0, flags=0):
    t = _times(times)
    n = t.shape[0]
    slots = np.zeros(n, SLOT_DT)
    res = Result()
    ev = np.zeros(MAX_EVENTS, dtype=[("kind", "<i4"), ("node", "<i4"), ("start", "<i8"), ("dur", "<i8")])
    nev = np.zeros(1, np.int32)
    _check(lib().orc_far(pid(profile), _ptr(_costs(costs)), _ptr(t), n, max_iterations, min_improvement_ppm, flags,
                         _ptr(slots), C.addressof(res), _ptr(ev), _ptr(nev)))
    return {"slots": slots, "result": res.asdict(), "events": ev[:nev[0]].copy()}


def refine(profile, costs, times, slots, makespan_in, max_iterations=100, min_improvement_ppm=0, flags=0):
    t = _times(times)
    n = t.shape[0]
    s = np.ascontiguousarray(slots, dtype=SLOT_DT).copy()
    res = Result()
    res.makespan_phase2 = makespan_in
    ev = np.zeros(MAX_EVENTS, dtype=[("kind", "<i4"), ("node", "<i4"), ("start", "<i8"), ("dur", "<i8")])
    nev = np.zeros(1, np.int32)
    _check(lib().orc_refine(pid(profile), _ptr(_costs(costs)), _ptr(t), n, max_iterations, min_improvement_ppm,
                            flags, _ptr(s), C.addressof(res), _ptr(ev), _ptr(nev)))
    return {"slots": s, "result": res.asdict(), "events": ev[:nev[0]].copy()}


def bruteforce(profile, times):
    t = _times(times)
    v = lib().orc_bruteforce(pid(profile), _ptr(t), t.shape[0])
    if v < 0:
        raise OracleError(v)
    return int(v)


def validate(profile, costs, times, slots, events, flags=0):
    t = _times(times)
    s = np.ascontiguousarray(slots, dtype=SLOT_DT)
    e = np.ascontiguousarray(events)
    return lib().orc_validate_flags(pid(profile), _ptr(_costs(costs)), _ptr(t), t.shape[0], _ptr(s), _ptr(e), len(e),
                                    flags)


def lower_bound(profile, times):
    t = _times(times)
    w = np.zeros(1, np.int64)
    h = np.zeros(1, np.int64)
    _check(lib().orc_lower_bound(pid(profile), _ptr(t), t.shape[0], _ptr(w), _ptr(h)))
    return int(w[0]), int(h[0])


def far_many(profile, costs, times, max_iterations=100, min_improvement_ppm=0, flags=0):
    """Sequential (single-thread) oracle over [I][n][|C|]; returns (makespans, results)."""
    t = _times(times)
    I, n = t.shape[0], t.shape[1]
    ms = np.zeros(I, np.int64)
    res = np.zeros(I, RESULT_DT)
    lib().orc_far_many(pid(profile), _ptr(_costs(costs)), _ptr(t), I, n, max_iterations, min_improvement_ppm, flags,
                       _ptr(ms), _ptr(res))
    return ms, res


def _far_many_worker(args):
    profile, costs, times, kw = args
    return far_many(profile, costs, times, **kw)


def _far_many_check_worker(args):
    """Solve a chunk with schedules and compare them with the given device slots (node, size_used,
    start) -> (makespans, results, number of instances whose schedule differs, first such index)."""
    profile, costs, times, dev_slots, kw = args
    t = _times(times)
    I, n = t.shape[0], t.shape[1]
    ms = np.zeros(I, np.int64)
    res = np.zeros(I, RESULT_DT)
    sl = np.zeros((I, n), SLOT_DT)
    lib().orc_far_many_slots(pid(profile), _ptr(_costs(costs)), _ptr(t), I, n, kw.get("max_iterations", 100),
                             kw.get("min_improvement_ppm", 0), kw.get("flags", 0), _ptr(ms), _ptr(res), _ptr(sl))
    bad = ((sl["node"] != dev_slots["node"]) | (sl["size_used"] != dev_slots["size_used"]) |
           (sl["start"] != dev_slots["start"])).any(axis=1)
    nb = int(bad.sum())
    return ms, res, nb, int(np.argmax(bad)) if nb else -1


def far_many_parallel(profile, costs, times, workers=None, **kw):
    """Oracle fanned out over host cores (independent processes) — for full parity only."""
    import concurrent.futures as cf
    t = _times(times)
    workers = workers or (os.cpu_count() or 1)
    if workers <= 1 or t.shape[0] < 64:
        return far_many(profile, costs, t, **kw)
    parts = np.array_split(np.arange(t.shape[0]), workers * 4)
    ms = np.zeros(t.shape[0], np.int64)
    res = np.zeros(t.shape[0], RESULT_DT)
    with cf.ProcessPoolExecutor(workers) as ex:
        futs = {ex.submit(_far_many_worker, (profile, costs, t[p[0]:p[-1] + 1], kw)): p for p in parts if len(p)}
        for f in cf.as_completed(futs):
            p = futs[f]
            m, r = f.result()
            ms[p[0]:p[-1] + 1] = m
            res[p[0]:p[-1] + 1] = r
    return ms, res


def far_many_parallel_check(profile, costs, times, dev_slots, workers=None, **kw):
    """Oracle over host cores with every schedule compared, chunk by chunk inside the workers, with
    the device slots dev_slots [I][n] (fields node, size_used, start) -> (makespans, results,
    number of mismatching schedules, first mismatching instance or -1)."""
    import concurrent.futures as cf
    t = _times(times)
    workers = workers or (os.cpu_count() or 1)
    parts = np.array_split(np.arange(t.shape[0]), max(1, workers * 8))
    ms = np.zeros(t.shape[0], np.int64)
    res = np.zeros(t.shape[0], RESULT_DT)
    nbad, first = 0, -1
    with cf.ProcessPoolExecutor(workers) as ex:
        futs = {ex.submit(_far_many_check_worker, (profile, costs, t[p[0]:p[-1] + 1],
                                                   dev_slots[p[0]:p[-1] + 1], kw)): p for p in parts if len(p)}
        for f in cf.as_completed(futs):
            p = futs[f]
            m, r, nb, fb = f.result()
            ms[p[0]:p[-1] + 1] = m
            res[p[0]:p[-1] + 1] = r
            if nb:
                nbad += nb
                g = p[0] + fb
                first = g if first < 0 else min(first, g)
    return ms, res, nbad, first


def stream(profile, costs, times, max_iterations=100, min_improvement_ppm=0, flags=0, ends=False):
    """§4 multi-batch fold over one stream: times [B][n][|C|].  Returns dict with makespan,
    trivial makespan, offsets [B], seam [B][4] {reversed, moves, swaps, reused}, slots [B][n]
    (batch-relative starts of the final timeline), per-batch results and the number of
    violations of the concatenated timeline's validator."""
    t = _times(times)
    B, n = t.shape[0], t.shape[1]
    out2 = np.zeros(2, np.int64)
    offs = np.zeros(B, np.int64)
    seam = np.zeros((B, 4), np.int32)
    slots = np.zeros((B, n), SLOT_DT)
    res = np.zeros(B, RESULT_DT)
    viol = np.zeros(1, np.int32)
    e = np.zeros(B, np.int64)
    if ends:  # + per-batch end O_k + E_k of the placed timeline (test entry orc_stream_ends)
        _check(lib().orc_stream_ends(pid(profile), _ptr(_costs(costs)), _ptr(t), B, n, max_iterations,
                                     min_improvement_ppm, flags, _ptr(out2), _ptr(offs), _ptr(seam), _ptr(slots),
                                     _ptr(res), _ptr(viol), _ptr(e)))
    else:
        _check(lib().orc_stream(pid(profile), _ptr(_costs(costs)), _ptr(t), B, n, max_iterations, min_improvement_ppm,
                                flags, _ptr(out2), _ptr(offs), _ptr(seam), _ptr(slots), _ptr(res), _ptr(viol)))
    out = {"makespan": int(out2[0]), "trivial": int(out2[1]), "offsets": offs, "seam": seam, "slots": slots,
           "results": res, "violations": int(viol[0])}
    if ends:
        out["ends"] = e
    return out


def stream_probe(profile, costs, times, k, delta):
    """(seam offset of batch k, violations of batches 0..k with batch k placed delta ticks early)."""
    t = _times(times)
    B, n = t.shape[0], t.shape[1]
    off = np.zeros(1, np.int64)
    viol = np.zeros(1, np.int32)
    _check(lib().orc_stream_probe(pid(profile), _ptr(_costs(costs)), _ptr(t), B, n, k, delta, _ptr(off), _ptr(viol)))
    return int(off[0]), int(viol[0])


def table_stats(profile, costs, tables, max_iterations=100, min_improvement_ppm=0, flags=0):
    """The evaluation statistics of PAPER.md §6 as exact fractions over a set of instances:
      rho   = omega / baseline, baseline = sum_i min_s s * t_i(s) / #slices   (Table 4)
      p_ref = (omega_no_ref / omega_ref - 1) * 100                             (Table 6)
    with omega_no_ref = FAR without phase 3 = the phase-2 makespan (R13), and the mean numbers of
    moves and swaps (Table 6).  Returns {"rho", "p_ref", "moves", "swaps", "count"} (Fractions)."""
    from fractions import Fraction
    t = np.asarray(tables, dtype=np.int32)
    ms, res = far_many(profile, costs, t, max_iterations=max_iterations, min_improvement_ppm=min_improvement_ppm,
                       flags=flags)
    S = lib().orc_num_slices(pid(profile))
    I = t.shape[0]
    rho = Fraction(0)
    pref = Fraction(0)
    for i in range(I):
        w, _ = lower_bound(profile, t[i])
        rho += Fraction(int(ms[i]) * S, w)
        pref += (Fraction(int(res["makespan_phase2"][i]), int(ms[i])) - 1) * 100
    return {"rho": rho / I, "p_ref": pref / I, "moves": Fraction(int(res["moves"].sum()), I),
            "swaps": Fraction(int(res["swaps"].sum()), I), "count": I}



def concat_stats(profile, costs, streams, max_iterations=100):
    """Tables 7 and 8: over streams of batches [S][B][n][|C|], the means of
      p_rev      = (omega_trivial / omega_rev - 1) * 100        reversal + seam offset only
      p_move/swap = (omega_trivial / omega_move/swap - 1) * 100  + seam moves and swaps
    and of the seam moves and swaps per stream, as exact Fractions."""
    from fractions import Fraction
    t = np.asarray(streams, dtype=np.int32)
    S = t.shape[0]
    prev = pms = Fraction(0)
    mv = sw = 0
    for s in range(S):
        full = stream(profile, costs, t[s], max_iterations=max_iterations)
        rev = stream(profile, costs, t[s], max_iterations=max_iterations, flags=NO_SEAM_MOVES)
        assert rev["trivial"] == full["trivial"]
        prev += (Fraction(full["trivial"], rev["makespan"]) - 1) * 100
        pms += (Fraction(full["trivial"], full["makespan"]) - 1) * 100
        mv += int(full["seam"][:, 1].sum())
        sw += int(full["seam"][:, 2].sum())
    return {"p_rev": prev / S, "p_move_swap": pms / S, "moves": Fraction(mv, S), "swaps": Fraction(sw, S), "count": S}


def multi_batch_p(profile, costs, batches, max_iterations=100):
    """Table 9: p_multi = (omega_multi / baseline_multi - 1) * 100 for one stream
    [B][n][|C|], baseline_multi = sum over all tasks of min_s s * t(s) / #slices (exact Fraction)."""
    from fractions import Fraction
    t = np.asarray(batches, dtype=np.int32)
    o = stream(profile, costs, t, max_iterations=max_iterations)
    W = sum(lower_bound(profile, t[k])[0] for k in range(t.shape[0]))
    S = lib().orc_num_slices(pid(profile))
    return (Fraction(o["makespan"] * S, W) - 1) * 100
