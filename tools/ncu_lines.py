"""Summarise an ncu --page source --print-source cuda,sass CSV: per source line stall samples and
instructions executed (top N).  Usage: python tools_ncu_lines.py file.csv [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, out, hdr = None, [], None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if not r or not hdr or r[0] == "" or r[0] == "Function Name":
        continue
    try:
        d = dict(zip(hdr[2:], r[2:]))
        samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        inst = int(d.get("Instructions Executed", "0") or 0)
        th = int(d.get("Thread Instructions Executed", "0") or 0)
    except ValueError:
        continue
    out.append((samp, inst, th, fname, r[0], r[1][:90]))
tot = sum(o[0] for o in out) or 1
toti = sum(o[1] for o in out) or 1
print(f"total samples {tot}  warp-inst {toti}")
for s, i, th, f, ln, src in sorted(out, reverse=True)[:N]:
    print(f"{100*s/tot:5.1f}% smp {100*i/toti:5.1f}% inst thr/inst {th/max(i,1):5.1f}  {f}:{ln}  {src}")
