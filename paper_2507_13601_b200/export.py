"""Schedule export: a FAR schedule plus its reconfiguration events as a
JSON document and as an SVG Gantt chart, and back.

The paper extracts the reconfiguration information "together with the obtained schedule" by a
BFS traversal of the output tree and executes it with Alg. 3 (out of
scope here: it needs MIG hardware).  This module is the host-side I/O around the device outputs:

* the schedule: per-task slots (``far_task_slot``: node, size used, start) from
  ``Far.solve_many`` / ``Far.schedule_batch``;
* the reconfiguration events: ``far_event`` records (create / destroy, node, start, duration)
  from ``Far.schedule_events`` (the line-26 replay of the schedule's node lists on the GPU,
  DESIGN.md R28);
* the tree: ``Far.node_table()`` (slice interval and parent of every node, include/far.h).

Nothing here computes any part of FAR: it only re-labels what the kernels returned (task end =
start + the runtime at the size used, read from the input table) and writes text.  Times are
integer ticks (1 tick = 1 ms with the Table 2 costs, R5).

JSON document (``schema`` = ``far-schedule/1``)::

  {"schema": "far-schedule/1", "profile": "A100", "tick_ms": 1, "makespan": int,
   "nodes":  [{"id", "slices": [lo, hi), "parent"}...],
   "tasks":  [{"task", "node", "size", "slices": [lo, hi), "start", "end"}...],     # task order
   "reconfigurations": [{"kind": "create"|"destroy", "node", "slices", "start", "end"}...]}  # start order
"""
from __future__ import annotations

import json

import numpy as np

SCHEMA = "far-schedule/1"
KINDS = ("create", "destroy")

SLOT_DT = np.dtype([("node", "u1"), ("size_used", "u1"), ("pad", "u1", 2), ("start", "<i4")])
EVENT_DT = np.dtype([("kind", "<i4"), ("node", "<i4"), ("start", "<i4"), ("dur", "<i4")])


def to_doc(profile, sizes, node_table, times, slots, events, makespan=None):
    """Build the JSON-able document of one schedule.

    profile: name; sizes: the profile's sizes in size-index order (``Far.sizes``);
    node_table: (lo, hi, parent) arrays (``Far.node_table()``); times: int [n][nsizes];
    slots: SLOT_DT-like records (fields node, size_used, start) [n]; events: EVENT_DT-like
    records (kind 0 create / 1 destroy, node, start, dur) [nev]; makespan: optional check value
    (the last task end is used and, if given, must equal it)."""
    lo, hi, par = (np.asarray(a) for a in node_table)
    t = np.asarray(times)
    size_index = {int(s): i for i, s in enumerate(sizes)}
    tasks = []
    end_max = 0
    for j in range(len(slots)):
        v = int(slots[j]["node"])
        sz = int(slots[j]["size_used"])
        st = int(slots[j]["start"])
        end = st + int(t[j, size_index[sz]])
        end_max = max(end_max, end)
        tasks.append({"task": j, "node": v, "size": sz, "slices": [int(lo[v]), int(hi[v])], "start": st, "end": end})
    if makespan is not None and int(makespan) != end_max:
        raise ValueError(f"makespan {makespan} != last task end {end_max}")
    recs = []
    for e in sorted((tuple(int(x) for x in (ev["start"], ev["node"], ev["kind"], ev["dur"])) for ev in events)):
        st, v, kind, dur = e
        recs.append({"kind": KINDS[kind], "node": v, "slices": [int(lo[v]), int(hi[v])], "start": st,
                     "end": st + dur})
    nodes = [{"id": v, "slices": [int(lo[v]), int(hi[v])], "parent": int(par[v])} for v in range(len(lo))]
    return {"schema": SCHEMA, "profile": profile, "tick_ms": 1, "makespan": end_max, "nodes": nodes,
            "tasks": tasks, "reconfigurations": recs}


def dumps(doc, **kw) -> str:
    return json.dumps(doc, **kw)


def loads(text: str) -> dict:
    doc = json.loads(text)
    if doc.get("schema") != SCHEMA:
        raise ValueError(f"not a {SCHEMA} document")
    return doc


def from_doc(doc):
    """-> (slots SLOT_DT [n], events EVENT_DT [nev]) exactly as the device returned them
    (events in start order)."""
    tasks = sorted(doc["tasks"], key=lambda x: x["task"])
    slots = np.zeros(len(tasks), SLOT_DT)
    for j, x in enumerate(tasks):
        if x["task"] != j:
            raise ValueError("task ids must be 0..n-1")
        slots[j]["node"] = x["node"]
        slots[j]["size_used"] = x["size"]
        slots[j]["start"] = x["start"]
    ev = np.zeros(len(doc["reconfigurations"]), EVENT_DT)
    for i, r in enumerate(doc["reconfigurations"]):
        ev[i]["kind"] = KINDS.index(r["kind"])
        ev[i]["node"] = r["node"]
        ev[i]["start"] = r["start"]
        ev[i]["dur"] = r["end"] - r["start"]
    return slots, ev


def gantt_svg(doc, width=1200, row=22, label=56) -> str:
    """SVG Gantt chart: one row per MIG slice, a task drawn across the slices of its instance,
    reconfigurations hatched (create) / grey (destroy)."""
    nsl = max(n["slices"][1] for n in doc["nodes"])
    span = max(1, max([doc["makespan"]] + [r["end"] for r in doc["reconfigurations"]]))
    sx = (width - label - 10) / span
    h = row * nsl + 40
    out = [f'<svg xmlns="http://www.w3.org/2000/svg" width="{width}" height="{h}" font-family="monospace" '
           f'font-size="10">',
           '<defs><pattern id="cr" width="6" height="6" patternUnits="userSpaceOnUse" '
           'patternTransform="rotate(45)"><rect width="3" height="6" fill="#d62728"/></pattern></defs>']
    for s in range(nsl):
        out.append(f'<text x="2" y="{20 + s * row + row * 0.65:.1f}">S{s}</text>')
        out.append(f'<line x1="{label}" y1="{20 + s * row}" x2="{width - 10}" y2="{20 + s * row}" stroke="#ddd"/>')

    def box(lo, hi, a, b, fill, title):
        x = label + a * sx
        w = max(0.5, (b - a) * sx)
        y = 20 + lo * row + 1
        return (f'<rect x="{x:.2f}" y="{y}" width="{w:.2f}" height="{(hi - lo) * row - 2}" fill="{fill}" '
                f'stroke="#333" stroke-width="0.3"><title>{title}</title></rect>')

    pal = ["#1f77b4", "#2ca02c", "#9467bd", "#8c564b", "#e377c2", "#17becf", "#bcbd22", "#ff7f0e"]
    for r in doc["reconfigurations"]:
        lo, hi = r["slices"]
        out.append(box(lo, hi, r["start"], r["end"], "url(#cr)" if r["kind"] == "create" else "#999",
                       f'{r["kind"]} node {r["node"]} [{r["start"]}, {r["end"]})'))
    for x in doc["tasks"]:
        lo, hi = x["slices"]
        out.append(box(lo, hi, x["start"], x["end"], pal[x["task"] % len(pal)],
                       f'task {x["task"]} size {x["size"]} node {x["node"]} [{x["start"]}, {x["end"]})'))
    out.append(f'<text x="{label}" y="{h - 6}">{doc["profile"]}: makespan {doc["makespan"]} ticks, '
               f'{len(doc["tasks"])} tasks, {len(doc["reconfigurations"])} reconfigurations</text>')
    out.append("</svg>")
    return "\n".join(out)
