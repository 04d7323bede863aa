"""Evaluation statistics of PAPER.md §6 from GPU outputs.

The per-instance quantities are the CUDA path's integer outputs -- makespan, phase-2 makespan,
moves, swaps (far_solve_many) and sum_i min_s s * t_i(s) (far_lower_bounds) -- so the means are
computed exactly (fractions) on the host:
  rho   = omega / baseline, baseline = sum_i min_s s * t_i(s) / #slices   (Table 4)
  p_ref = (omega_no_ref / omega_ref - 1) * 100                             (Table 6)
omega_no_ref is FAR without phase 3, i.e. the phase-2 makespan of the same run (R13).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np


def table_means(nslices: int, makespan, makespan_phase2, moves, swaps, sum_min_work) -> dict:
    """Exact means over instances (numpy integer arrays) -> {"rho", "p_ref", "moves", "swaps", "count"}."""
    ms = np.asarray(makespan, dtype=np.int64)
    m2 = np.asarray(makespan_phase2, dtype=np.int64)
    w = np.asarray(sum_min_work, dtype=np.int64)
    I = len(ms)
    rho = sum((Fraction(int(a) * nslices, int(b)) for a, b in zip(ms, w)), Fraction(0))
    pref = sum(((Fraction(int(b), int(a)) - 1) * 100 for a, b in zip(ms, m2)), Fraction(0))
    return {"rho": rho / I, "p_ref": pref / I, "moves": Fraction(int(np.sum(moves)), I),
            "swaps": Fraction(int(np.sum(swaps)), I), "count": I}


def solve_and_measure(F, d_times, **kw) -> dict:
    """far_solve_many + far_lower_bounds on device-resident tables, then table_means."""
    from . import far
    ms, _, rs = F.solve_many(d_times, sched=False, **kw)
    w, _ = F.lower_bounds(d_times)
    res = far.results_np(rs)
    return table_means(F.nslices, ms.cpu().numpy(), res["makespan_phase2"], res["moves"], res["swaps"],
                       w.cpu().numpy())


def concat_means(F, d_streams, **kw) -> dict:
    """Tables 7 and 8 from far_concat_streams on device-resident streams
    [S][B][n][|C|]: means over streams of p_rev (reversal + seam offset only, FAR_NO_SEAM_MOVES),
    p_move/swap (the full fold) against the trivial concatenation, and of the seam moves / swaps."""
    from . import far
    flags = kw.pop("flags", 0)
    sm, _, _, _, se = F.concat_streams(d_streams, sched=False, batch_res=False, flags=flags, **kw)
    sr, _, _, _, _ = F.concat_streams(d_streams, sched=False, batch_res=False, seam=False,
                                      flags=flags | far.NO_SEAM_MOVES, **kw)
    sm, sr, se = sm.cpu().numpy(), sr.cpu().numpy(), se.cpu().numpy()
    S = sm.shape[0]
    assert (sm[:, 1] == sr[:, 1]).all()
    prev = sum(((Fraction(int(a), int(b)) - 1) * 100 for a, b in zip(sm[:, 1], sr[:, 0])), Fraction(0))
    pms = sum(((Fraction(int(a), int(b)) - 1) * 100 for a, b in zip(sm[:, 1], sm[:, 0])), Fraction(0))
    return {"p_rev": prev / S, "p_move_swap": pms / S, "moves": Fraction(int(se[:, :, 1].sum()), S),
            "swaps": Fraction(int(se[:, :, 2].sum()), S), "count": S}


def multi_batch_p(F, d_batches, **kw) -> Fraction:
    """Table 9: p_multi = (omega_multi / baseline_multi - 1) * 100 of one stream
    [B][n][|C|] (far_concat_streams + far_lower_bounds, exact)."""
    sm, _, _, _, _ = F.concat_streams(d_batches[None].contiguous(), sched=False, batch_res=False, seam=False, **kw)
    w, _ = F.lower_bounds(d_batches)
    W = int(w.sum().item())
    return (Fraction(int(sm[0, 0].item()) * F.nslices, W) - 1) * 100
