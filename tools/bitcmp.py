"""Save L / tau / pivots of a few factorizations (library chosen by SKEWLTL_B200_LIB)
to argv[1]; with argv[2] also given, compare the two files bit for bit."""
import sys
import numpy as np
sys.path.insert(0, ".")
if len(sys.argv) > 2:
    a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
    bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
    print("BITCMP", "identical" if not bad else f"DIFFER {bad}")
    sys.exit(0)
import paper_2411_09859_b200 as pk
from paper_2411_09859_b200.inputs import skew_lower
out = {}
for n, b in ((4096, 128), (512, 512), (2000, 96)):
    r = pk.ltlt_blk_piv(pk.SkewMatrixLower(skew_lower(n, 0)), b=b)
    out[f"L{n}"], out[f"t{n}"], out[f"p{n}"] = np.asarray(r.l.data), np.asarray(r.t.tau), np.asarray(r.p.pivots)
np.savez(sys.argv[1], **out)
