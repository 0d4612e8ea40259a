"""The multi-cluster panel (several co-resident 16-CTA clusters; used by the driver
above ~6K rows, e.g. config 3) forced at small n, against the oracle: pivots
bit-exact, L / tau within 1e-10 * n, at Q = 2 and Q = 3 clusters.  At these
sizes whole clusters run out of rows below the pivot column (the empty-cluster
record path of the leader exchange), which the config-3 run never reaches."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("q", [2, 3])
def test_forced_multi_cluster_panel(q):
    env = dict(os.environ, SKL_FORCE_MULTI="1", SKL_MULTI_Q=str(q))
    p = subprocess.run([sys.executable, str(ROOT / "tests" / "multi_worker.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "MULTI_OK" in p.stdout, p.stdout[-2000:] + p.stderr[-4000:]
