"""Aggregate the combined cuda,sass source export (see tools/ncu_src.py) by line ranges of one file.
Usage: python tools/ncu_src_regions.py file.csv far_kernel.cuh name:start name:start ..."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
target = sys.argv[2]
ranges = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[3:]]


def region(line):
    name = "pre"
    for nm, s in ranges:
        if line >= s:
            name = nm
    return name


agg, hdr, f = {}, None, None
for r in rows:
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not r or not hdr or not r[0].isdigit():
        continue
    d = dict(zip(hdr[4:], r[4:]))
    try:
        s = int(d["Warp Stall Sampling (All Samples)"] or 0)
        i = int(d["Instructions Executed"] or 0)
        t = int(d["Thread Instructions Executed"] or 0)
    except ValueError:
        continue
    k = region(int(r[0])) if f == target else "lib:" + f
    a = agg.setdefault(k, [0, 0, 0])
    a[0] += s
    a[1] += i
    a[2] += t
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:22s} samples {100 * v[0] / ts:5.1f}%  warp-inst {100 * v[1] / ti:5.1f}%  lanes/inst {v[2] / max(v[1], 1):5.1f}")
