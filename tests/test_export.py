"""NEXT-4 schedule export (paper_2507_13601_b200/export.py): JSON and Gantt of a schedule plus its
reconfiguration events ("a BFS traversal of the output tree allows to properly extract this
reconfiguration info together with the obtained schedule").  CPU tests: schedules and events
from the oracle are exported, parsed back and re-checked by the oracle's own validator (constraints
1-3); a corrupted document must fail it.  The GPU test (test_gpu_check.py style) exports
device outputs (far_solve_many + far_schedule_events)."""
import json
import xml.etree.ElementTree as ET

import numpy as np
import pytest

from oracle import oracle as O
from paper_2507_13601_b200 import export, inputs

SIZES = {"A30": [1, 2, 4], "A100": [1, 2, 3, 4, 7], "H100": [1, 2, 3, 4, 7]}


def oracle_case(profile, n, seed, zero=False):
    tab = inputs.synthetic(profile, n, 1, seed)[0]
    costs = inputs.reconfig_costs(profile, zero=zero)
    out = O.far(profile, costs, tab)
    return tab, costs, out


def doc_of(profile, tab, out):
    lo, hi, par = O.nodes(profile)
    return export.to_doc(profile, SIZES[profile], (lo, hi, par), tab, out["slots"], out["events"],
                         makespan=out["result"]["makespan"])


def back_to_oracle(slots, ev):
    s = np.zeros(len(slots), O.SLOT_DT)
    s["node"], s["size_used"], s["start"] = slots["node"], slots["size_used"], slots["start"]
    e = np.zeros(len(ev), dtype=[("kind", "<i4"), ("node", "<i4"), ("start", "<i8"), ("dur", "<i8")])
    for k in ("kind", "node", "start", "dur"):
        e[k] = ev[k]
    return s, e


@pytest.mark.parametrize("profile,n,seed", [("A30", 8, 1), ("A30", 40, 2), ("A100", 16, 3), ("A100", 64, 4),
                                            ("H100", 33, 5)])
def test_roundtrip_validates(profile, n, seed):
    tab, costs, out = oracle_case(profile, n, seed)
    doc = doc_of(profile, tab, out)
    text = export.dumps(doc)
    doc2 = export.loads(text)
    assert doc2 == json.loads(json.dumps(doc))
    slots, ev = export.from_doc(doc2)
    assert (slots["node"] == out["slots"]["node"]).all() and (slots["start"] == out["slots"]["start"]).all()
    assert (slots["size_used"] == out["slots"]["size_used"]).all()
    assert len(ev) == len(out["events"])
    s, e = back_to_oracle(slots, ev)
    assert O.validate(profile, costs, tab, s, e) == 0
    # document invariants: task end = start + t at the size used; reconfigurations disjoint in time
    for x in doc["tasks"]:
        assert x["end"] - x["start"] == tab[x["task"], SIZES[profile].index(x["size"])]
    recs = doc["reconfigurations"]
    assert all(recs[i]["end"] <= recs[i + 1]["start"] for i in range(len(recs) - 1))
    assert doc["makespan"] == out["result"]["makespan"] == max(x["end"] for x in doc["tasks"])


def test_corrupted_document_fails_validation():
    profile = "A100"
    tab, costs, out = oracle_case(profile, 24, 7)
    doc = doc_of(profile, tab, out)
    # move the task that starts last on its node to start together with another task on its node
    by_node = {}
    for x in doc["tasks"]:
        by_node.setdefault(x["node"], []).append(x)
    node, xs = next((v, xs) for v, xs in by_node.items() if len(xs) >= 2)
    xs.sort(key=lambda x: x["start"])
    xs[-1]["start"] = xs[0]["start"]
    slots, ev = export.from_doc(doc)
    s, e = back_to_oracle(slots, ev)
    assert O.validate(profile, costs, tab, s, e) > 0
    # and a reconfiguration overlapping another one
    doc = doc_of(profile, tab, out)
    if len(doc["reconfigurations"]) >= 2:
        doc["reconfigurations"][1]["start"] = doc["reconfigurations"][0]["start"]
        slots, ev = export.from_doc(doc)
        s, e = back_to_oracle(slots, ev)
        assert O.validate(profile, costs, tab, s, e) > 0


def test_gantt_svg_well_formed():
    tab, costs, out = oracle_case("A100", 16, 11)
    doc = doc_of("A100", tab, out)
    svg = export.gantt_svg(doc)
    root = ET.fromstring(svg)
    rects = [el for el in root.iter() if el.tag.endswith("rect")]
    # one rect per task and per reconfiguration (+ the hatch pattern's)
    assert len(rects) == len(doc["tasks"]) + len(doc["reconfigurations"]) + 1


def test_bad_makespan_rejected():
    tab, costs, out = oracle_case("A30", 8, 3)
    lo, hi, par = O.nodes("A30")
    with pytest.raises(ValueError):
        export.to_doc("A30", SIZES["A30"], (lo, hi, par), tab, out["slots"], out["events"],
                      makespan=out["result"]["makespan"] + 1)
    with pytest.raises(ValueError):
        export.loads(json.dumps({"schema": "other"}))


@pytest.mark.gpu
def test_gpu_outputs_export_and_validate():
    """Device schedules and device-extracted events (far_schedule_events) exported, parsed back and
    accepted by the oracle's validator; the document's makespan is the device makespan."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2507_13601_b200 import far
    for wname, count in (("M1", 40), ("M2", 40), ("M5", 8)):
        w = inputs.WORKLOADS[wname]
        tab = w.table(count=count)
        costs = w.costs()
        F = far.Far(w.profile, costs)
        d = torch.from_numpy(np.ascontiguousarray(tab)).to("cuda:0")
        ms, sd, _ = F.solve_many(d)
        ev, nev, _ = F.schedule_events(d, sd)
        torch.cuda.synchronize()
        F.sync()
        slots = far.slots_np(sd)
        evs = far.events_np(ev, nev)
        ms = ms.cpu().numpy()
        node_table = F.node_table()
        for i in range(count):
            doc = export.to_doc(w.profile, F.sizes, node_table, tab[i], slots[i], evs[i], makespan=ms[i])
            s2, e2 = export.from_doc(export.loads(export.dumps(doc)))
            s, e = back_to_oracle(s2, e2)
            assert O.validate(w.profile, costs, tab[i], s, e) == 0, (wname, i)
            assert doc["makespan"] == ms[i]
        F.close()
