"""The single-cluster panel's push mode (candidate rows by st.async, lazy
interchanges through position labels) performs the same arithmetic as the L2
row-exchange mode (SKL_PANEL_PUSH=0): L, tau and pivots must be bit-identical.
Both runs are also held to the oracle by test_gpu_blocked.py / test_gpu_twostep.py."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def run(tmp_path, push):
    out = tmp_path / f"push{push}.npz"
    env = dict(os.environ, SKL_PANEL_PUSH=str(push))
    p = subprocess.run([sys.executable, str(ROOT / "tests" / "push_worker.py"), str(out)], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "PUSH_OK" in p.stdout, p.stdout[-2000:] + p.stderr[-4000:]
    return np.load(out)


def test_push_mode_bit_identical_to_l2_exchange(tmp_path):
    a, b = run(tmp_path, 1), run(tmp_path, 0)
    assert sorted(a.files) == sorted(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
