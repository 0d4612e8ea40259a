"""CallTrace parity (reference instrument.py:44-54 and the record_call sites of
kernels2.py / kernels3.py).  The GPU drivers run fused kernels, so the trace
they hand to ``instrument.tracing`` is the reference's call sequence replayed
from the schedule and the returned tau / pivots -- the same replay that yields
the flop tallies.  Pinned against traces.json, recorded from the unmodified
reference (tests/golden/make_traces.py).  CPU tests feed the replay the
oracle's tau / pivots; the gpu test runs the product drivers under tracing."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2411_09859_b200 import instrument as ins
from paper_2411_09859_b200.inputs import skew_lower

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))
from trace_cases import TRACE_CASES, first_column_vec, run_case  # noqa: E402

GOLD = json.loads((HERE / "golden" / "traces.json").read_text())


def replay(kind, kw):
    n = kw["n"]
    x = skew_lower(n, kw["seed"])
    if kind == "blk_piv":
        o = oracle.ltlt_blk_piv(x, b=kw["b"], fused=kw["fused"])
        return ins.flops_blk_piv(n, kw["b"], kw["fused"], o.pivots, o.tau)
    if kind == "blk":
        o = oracle.ltlt_blk(x, kw["b"], kw["driver"], kw["pv"])
        return ins.flops_blk_unpivoted(n, kw["b"], kw["driver"], kw["pv"], o.tau, o.work)
    if kind == "unb_twostep":
        o = oracle.ltlt_unb_twostep(x, kw["pivot"])
        piv = o.pivots if kw["pivot"] else np.zeros(n, dtype=np.int64)
        return ins.flops_unb_twostep(n, piv, o.tau, pivot=kw["pivot"])
    if kind == "unb_ll":
        fc = first_column_vec(n) if kw.get("first_column") else None
        o = oracle.ltlt_unb_ll(x, kw["pivot"], fc)
        return ins.flops_unb_ll(n, o.tau, o.pivots if kw["pivot"] else None, first_column=fc is not None)
    if kind == "unb_rl":
        o = oracle.ltlt_unb_rl(x, kw["pivot"])
        return ins.flops_unb_rl(n, o.tau, o.pivots if kw["pivot"] else None)
    if kind == "unb_panel":
        o = oracle.ltlt_unb_panel(x, kw["width"], kw["variant"], kw["pivot"])
        piv = None
        if kw["pivot"]:
            piv = np.zeros(n, dtype=np.int64)
            piv[:len(o.pivots)] = o.pivots
        return ins.flops_unb_panel(n, kw["width"], kw["variant"], o.tau, piv)
    raise ValueError(kind)


@pytest.mark.parametrize("key,kind,kw", TRACE_CASES, ids=[c[0] for c in TRACE_CASES])
def test_replayed_trace_matches_reference(key, kind, kw):
    tr = ins.CallTrace()
    with ins.tracing(tr):
        fc = replay(kind, kw)
    assert [list(c) for c in tr.calls] == GOLD[key]["calls"]
    assert dict(level2=fc.level2, level3=fc.level3, panel=fc.panel, pivot=fc.pivot) == GOLD[key]["flops"]


def test_counting_and_scope_api():
    fc = ins.FlopCounter()
    tr = ins.CallTrace()
    with ins.counting(fc), ins.tracing(tr), ins.scope("panel"):
        assert ins.current_scope() == "panel"
        ins.record_call("skew_rank2")
        ins.add_flops("level2", 12)
    assert ins.current_scope() == "trailing"
    assert tr.count("skew_rank2", "panel") == 1 and tr.count(scope="trailing") == 0 and fc.level2 == 12
    ins.add_flops("level2", 5)  # no active counter: dropped
    assert fc.level2 == 12


def test_reference_trace_properties():
    # the reference's own TestTrace facts (tests/test_blocked.py:160-205), on the fixture
    m, b = 48, 8
    iters = (m - 1 + b - 1) // b
    var1 = ins.CallTrace([tuple(c) for c in GOLD["blk_var1_ll"]["calls"]])
    assert var1.count("skew_rank2", "trailing") == iters - 1
    for d in ("var2a", "var2b", "twostep"):
        assert ins.CallTrace([tuple(c) for c in GOLD[f"blk_{d}_ll"]["calls"]]).count("skew_rank2", "trailing") == 0
    rl = ins.CallTrace([tuple(c) for c in GOLD["blk_var2a_rl"]["calls"]])
    assert rl.count("skew_rank2", "trailing") == 0 and rl.count("skew_rank2", "panel") > 0


@pytest.mark.gpu
@pytest.mark.parametrize("key,kind,kw", TRACE_CASES, ids=[c[0] for c in TRACE_CASES])
def test_driver_trace_on_gpu(key, kind, kw):
    import paper_2411_09859_b200 as pk
    tr = ins.CallTrace()
    fc = ins.FlopCounter()
    with ins.tracing(tr), ins.counting(fc):
        r = run_case(pk, kind, kw, skew_lower)
    assert [list(c) for c in tr.calls] == GOLD[key]["calls"]
    assert r.flops == fc == pk.FlopCounter(**GOLD[key]["flops"])
