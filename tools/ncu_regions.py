"""Aggregate an ncu source CSV (--print-source cuda,sass) by line ranges.
Usage: python tools/ncu_regions.py file.csv name:start name:start ...   (ranges of far_kernel.cuh)"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
ranges = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[2:]]
def ph(l):
    n = "pre"
    for nm, s in ranges:
        if l >= s: n = nm
    return n
agg = {}; hdr = None; f = None
for r in rows:
    if r and r[0] == "File Path": f = r[1].split('/')[-1]; continue
    if r and r[0] == "Line No": hdr = r; continue
    if not r or not hdr or r[0] in ("", "Function Name"): continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0); i = int(d["Instructions Executed"] or 0)
        t = int(d["Thread Instructions Executed"] or 0)
    except Exception:
        continue
    k = ph(int(r[0])) if f == (sys.argv[0] and __import__("os").environ.get("NCU_FILE","far_kernel.cuh")) else "lib:" + f
    if k == "frontier": k = "frontier(p2)" if t / max(i, 1) > 4 else "frontier(lane0)"
    a = agg.setdefault(k, [0, 0, 0]); a[0] += s; a[1] += i; a[2] += t
ts = sum(v[0] for v in agg.values()); ti = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:22s} samples {100*v[0]/ts:5.1f}%  warp-inst {100*v[1]/ti:5.1f}%  lanes/inst {v[2]/max(v[1],1):5.1f}")
