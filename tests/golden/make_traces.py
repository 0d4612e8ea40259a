"""Record the reference's CallTrace (instrument.py:44-54, kernels' record_call
sites) for the cases in trace_cases.py by running the UNMODIFIED reference here:
    python tests/golden/make_traces.py   ->  tests/golden/traces.json"""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, str(HERE))

import skewltl  # noqa: E402
from skewltl import instrument  # noqa: E402

from paper_2411_09859_b200.inputs import skew_lower  # noqa: E402
from trace_cases import TRACE_CASES, run_case  # noqa: E402

out = {}
for key, kind, kw in TRACE_CASES:
    tr = instrument.CallTrace()
    with instrument.tracing(tr):
        r = run_case(skewltl, kind, kw, skew_lower)
    out[key] = {"calls": [list(c) for c in tr.calls],
                "flops": dict(level2=r.flops.level2, level3=r.flops.level3, panel=r.flops.panel, pivot=r.flops.pivot)}
(HERE / "traces.json").write_text(json.dumps(out, indent=0))
print(f"wrote {len(out)} traces")
