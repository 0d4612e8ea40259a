"""Output / exchange formats either side of the path:
Matrix Market I/O (mmio.py:18-71, host file formatting) on CPU, and the packed
factor layout pack_in_place / unpack_in_place (core.py:349-375, CUDA kernels)
on the GPU."""

import numpy as np
import pytest

import oracle
from conftest import GOLDEN
from paper_2411_09859_b200.inputs import skew_lower


def pk():
    import paper_2411_09859_b200 as m
    return m


def test_mm_write_matches_reference_bytes(tmp_path):
    x = skew_lower(9, 4)
    x[5, 2] = 0.0
    out = tmp_path / "x.mtx"
    pk().mm_write(out, pk().SkewMatrixLower(x))
    assert out.read_text() == (GOLDEN / "mm_small.mtx").read_text()


def test_mm_read_round_trip():
    x = pk().mm_read(GOLDEN / "mm_small.mtx")
    ref = skew_lower(9, 4)
    ref[5, 2] = 0.0
    assert np.array_equal(np.tril(x.data, -1), np.tril(ref, -1))


@pytest.mark.parametrize("text,msg", [
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n2 1 1.0\n", "symmetry qualifier"),
    ("%%MatrixMarket matrix array real skew-symmetric\n2 2\n", "unsupported format"),
    ("MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n2 1 1.0\n", "malformed"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n1 2 1.0\n", "above the diagonal"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n1 1 3.0\n", "nonzero diagonal"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 3 1\n2 1 1.0\n", "expected square"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 0\n2 1 1.0\n", "more entries"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 1\n3 1 1.0\n", "out of range"),
])
def test_mm_read_rejects(tmp_path, text, msg):
    p = tmp_path / "bad.mtx"
    p.write_text(text)
    with pytest.raises(ValueError, match=msg):
        pk().mm_read(p)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 2, 5, 130])
def test_pack_unpack_round_trip(n):
    x = skew_lower(n, n)
    r = pk().ltlt_blk_piv(pk().SkewMatrixLower(x), b=16)
    packed = pk().SkewMatrixLower(x.copy(order="F"))
    pk().pack_in_place(packed, r.l, r.t)
    # restated layout (core.py:357-362): tau on the subdiagonal, L below it
    want = x.copy(order="F")
    for j in range(n - 1):
        want[j + 1, j] = r.t.tau[j]
        want[j + 2:, j] = r.l.data[j + 2:, j]
    assert np.array_equal(packed.data, want)
    l2, t2 = pk().unpack_in_place(packed)
    assert np.array_equal(t2.tau, r.t.tau)
    assert np.array_equal(l2.dense(), r.l.dense())
    assert np.array_equal(np.triu(l2.data), np.zeros((n, n)))
