"""Summarise an `ncu -i X --page source --csv --print-source cuda,sass --launch-skip S --launch-count 1`
export (rows: CUDA line with its aggregate metrics, then its SASS rows).
Usage: python tools/ncu_src.py file.csv [N] [--stalls]
Prints the top-N CUDA lines by warp-stall samples, with warp-instructions and lanes/instruction,
and (with --stalls) the top stall reasons of each line."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
show_stalls = "--stalls" in sys.argv
fname, hdr, out = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or not hdr or not r[0].isdigit():
        continue
    d = dict(zip(hdr[4:], r[4:]))

    def g(k):
        try:
            return int(d.get(k, "0") or 0)
        except ValueError:
            return 0
    st = {k: g(k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}
    out.append((g("Warp Stall Sampling (All Samples)"), g("Instructions Executed"),
                g("Thread Instructions Executed"), fname, r[0], r[1][:80], st))
tot = sum(o[0] for o in out) or 1
toti = sum(o[1] for o in out) or 1
print(f"total samples {tot}  warp-inst {toti}")
for s, i, th, f, ln, src, st in sorted(out, key=lambda o: -o[0])[:N]:
    extra = ""
    if show_stalls:
        top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
        extra = "  [" + " ".join(f"{k[6:]}={100 * v / max(s, 1):.0f}%" for k, v in top if v) + "]"
    print(f"{100 * s / tot:5.1f}% smp {100 * i / toti:5.1f}% inst {th / max(i, 1):5.1f}/i {f}:{ln} {src.strip()}{extra}")
