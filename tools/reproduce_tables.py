"""Statistical reproduction of PAPER.md Tables 4, 6, 7, 8, 9 and the large-n scheduler-time workload on
the GPU, side by side with the values the paper prints
(tests/golden/paper_tables.json).  The inputs come from this repo's §6.3 generator,
not the paper's, so agreement is a plausibility signal for the readings, not a parity claim; the
parity claim is `--oracle`: every cell's exact means equal the CPU oracle's.

Usage (GPU box): python tools/reproduce_tables.py [--count 1000] [--oracle] [--out profiles/r1_tables]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2507_13601_b200 import far, inputs, stats  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=1000)
    ap.add_argument("--oracle", action="store_true", help="check every cell's means against the CPU oracle")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r1_tables"))
    args = ap.parse_args()
    import torch
    dev = torch.device("cuda:0")
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_tables.json")))
    costs = inputs.reconfig_costs("A100")
    F = far.Far("A100", costs)
    O = None
    if args.oracle:
        from oracle import oracle as O
        O.build()
    out = {"count": args.count, "table4": {}, "table6": {}, "table7_8": {}, "table9": {}, "large_n": {},
           "oracle_checked": bool(args.oracle)}

    def cell(n, scaling, times, seed):
        tab = inputs.synthetic("A100", n, args.count, seed, scaling=scaling, times=times)
        got = stats.solve_and_measure(F, torch.from_numpy(tab).to(dev))
        F.sync()
        if O is not None:
            assert got == O.table_stats("A100", costs, tab), (n, scaling, times)
        return got

    t4 = gold["table4_rho_A100_wide"]
    for sc in ("poor", "mixed", "good"):
        rows = []
        for n, paper in zip(t4["n"], t4[sc]):
            g = cell(n, sc, "wide", 4000 + n)
            rows.append({"n": n, "rho": float(g["rho"]), "paper": paper})
        out["table4"][sc] = rows
    t6 = gold["table6_refinement_A100"]
    for sc in ("poor", "mixed", "good"):
        for tm in ("narrow", "wide"):
            rows = []
            for n, paper in zip(t6["n"], t6[f"{sc}_{tm}"]):
                g = cell(n, sc, tm, 6000 + n)
                rows.append({"n": n, "p_ref": float(g["p_ref"]), "moves": float(g["moves"]), "swaps": float(g["swaps"]),
                             "paper": paper})
            out["table6"][f"{sc}_{tm}"] = rows
    # Tables 7 and 8: concatenations of two FAR schedules (the second reversed; the paper reports
    # both orders together and finds them alike), count pairs per cell
    t7, t8 = gold["table7_concat_A100"], gold["table8_concat_moves_swaps_A100"]
    for sc in ("poor", "mixed", "good"):
        for tm in ("narrow", "wide"):
            rows = []
            for q, n in enumerate(t7["n"]):
                tab = inputs.synthetic("A100", n, 2 * args.count, 7000 + n, scaling=sc, times=tm).reshape(
                    args.count, 2, n, -1)
                g = stats.concat_means(F, torch.from_numpy(tab).to(dev))
                F.sync()
                if O is not None:
                    assert g == O.concat_stats("A100", costs, tab), (n, sc, tm)
                rows.append({"n": n, "p_rev": float(g["p_rev"]), "p_move_swap": float(g["p_move_swap"]),
                             "moves": float(g["moves"]), "swaps": float(g["swaps"]),
                             "paper7": t7[f"{sc}_{tm}"][q], "paper8": t8[f"{sc}_{tm}"][q]})
            out["table7_8"][f"{sc}_{tm}"] = rows
    # Table 9: one stream of 1001 batches per cell, WideTimes
    t9 = gold["table9_multibatch_A100_wide"]
    for sc in ("poor", "mixed", "good"):
        rows = []
        for n, paper in zip(t9["n"], t9[sc]):
            tab = inputs.synthetic("A100", n, 1001, 9100 + n, scaling=sc, times="wide")
            g = stats.multi_batch_p(F, torch.from_numpy(tab).to(dev))
            F.sync()
            if O is not None:
                assert g == O.multi_batch_p("A100", costs, tab), (n, sc)
            rows.append({"n": n, "p_multi": float(g), "paper": paper})
        out["table9"][sc] = rows
    # the paper's scheduler-time workload: 1000 instances, MixedScaling, n = 100 / 500 / 1000
    ln = gold["large_n_cpu_ms"]
    for n, paper_ms in zip(ln["n"], ln["ms"]):
        tab = inputs.synthetic("A100", n, args.count, 9000 + n)
        d = torch.from_numpy(tab).to(dev)
        F.solve_many(d, sched=False)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            F.solve_many(d, sched=False)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        out["large_n"][str(n)] = {"gpu_ms_for_all": ms, "gpu_us_per_instance": 1000.0 * ms / args.count,
                                  "paper_cpu_ms_per_instance": paper_ms}
    with open(args.out + ".json", "w") as f:
        json.dump(out, f, indent=1)
    lines = ["# Statistical reproduction of PAPER.md Tables 4 and 6 on the GPU (NEXT-1)", "",
             f"{args.count} instances per cell, this repo's §6.3 generator (DESIGN.md §5), Table 2 A100 costs, "
             f"1 ms ticks.  Means computed exactly from the CUDA path's integer outputs (`stats.py`)"
             + ("; every cell equal to the CPU oracle's exact means." if args.oracle else "."), "",
             "## Table 4: mean rho = omega / baseline, A100, WideTimes (ours / paper)", "",
             "| scaling | " + " | ".join(f"n={r['n']}" for r in out["table4"]["poor"]) + " |",
             "|---|" + "---|" * len(out["table4"]["poor"])]
    for sc, rows in out["table4"].items():
        lines.append(f"| {sc} | " + " | ".join(f"{r['rho']:.3f} / {r['paper']:.2f}" for r in rows) + " |")
    lines += ["", "## Table 6: mean p_ref (%), moves, swaps (ours / paper)", "",
              "| workload | " + " | ".join(f"n={r['n']}" for r in out["table6"]["poor_narrow"]) + " |",
              "|---|" + "---|" * len(out["table6"]["poor_narrow"])]
    for k, rows in out["table6"].items():
        lines.append(f"| {k} | " + " | ".join(
            f"{r['p_ref']:.2f}, {r['moves']:.2f}, {r['swaps']:.2f} / {r['paper'][0]:.2f}, {r['paper'][1]:.2f}, "
            f"{r['paper'][2]:.2f}" for r in rows) + " |")
    lines += ["", "## Tables 7 and 8: concatenation of two FAR schedules, p_rev / p_move/swap (%) and seam moves, swaps "
              "(ours / paper)", "",
              "| workload | " + " | ".join(f"n={r['n']}" for r in out["table7_8"]["poor_narrow"]) + " |",
              "|---|" + "---|" * len(out["table7_8"]["poor_narrow"])]
    for k, rows in out["table7_8"].items():
        lines.append(f"| {k} | " + " | ".join(
            f"{r['p_rev']:.2f}, {r['p_move_swap']:.2f}; {r['moves']:.2f}, {r['swaps']:.2f} / "
            f"{r['paper7'][0]:.2f}, {r['paper7'][1]:.2f}; {r['paper8'][0]:.2f}, {r['paper8'][1]:.2f}" for r in rows) + " |")
    lines += ["", "## Table 9: p_multi-batch (%), 1001 batches, WideTimes (ours / paper)", "",
              "| scaling | " + " | ".join(f"n={r['n']}" for r in out["table9"]["poor"]) + " |",
              "|---|" + "---|" * len(out["table9"]["poor"])]
    for sc, rows in out["table9"].items():
        lines.append(f"| {sc} | " + " | ".join(f"{r['p_multi']:.2f} / {r['paper']:.2f}" for r in rows) + " |")
    lines += ["", "## Scheduler time at large n (MixedScaling; paper: C++ on a Ryzen 5 4600H, one batch at a time)", "",
              "| n | GPU, all instances (ms) | GPU per instance (us) | paper per instance (ms) |", "|---|---|---|---|"]
    for n, r in out["large_n"].items():
        lines.append(f"| {n} | {r['gpu_ms_for_all']:.2f} | {r['gpu_us_per_instance']:.2f} | {r['paper_cpu_ms_per_instance']} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
