"""CPU: host-side logic, the C-ABI library surface, closed-form flop counts."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
from conftest import ROOT, worked_example
from paper_2411_09859_b200 import _capi
from paper_2411_09859_b200.core import (InvalidVariant, PermutationVector, SkewMatrixLower, SkewTridiagonal,
                                        UnitLowerFactor, ZeroPivot, compose_permutation, form_s_splitting)
from paper_2411_09859_b200.inputs import CONFIGS, config_input, skew_lower
from paper_2411_09859_b200.instrument import (FlopCounter, flops_blk_piv, flops_unb_twostep,
                                              reference_schedule)

HEADER = ROOT / "include" / "skewltl_b200.h"


def header_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(skl_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _capi.load()
    names = header_functions()
    assert len(names) >= 17
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_capi.SIGNATURES)


def test_library_version_and_no_compute_without_gpu():
    lib = _capi.load()
    assert b"sm_100a" in lib.skl_version()
    # workspace queries are pure host logic; safe without a device
    assert lib.skl_skr2k_workspace_size(4096, 128) > 0
    assert lib.skl_sktri_rankk_workspace_size(100, 8) > 0


def test_bad_arguments_rejected_before_any_launch():
    lib = _capi.load()
    # negative sizes / short leading dimensions are caught on the host
    assert lib.skl_skr2k_lower(-1, 2, 1.0, None, 1, None, 1, 1.0, None, 1, 1, None, 0, None, None) == _capi.SKL_BAD_ARGUMENT
    assert lib.skl_ltlt_blk_piv(8, 4, 7, None, 8, None, 8, None, None, None, 0, None) == _capi.SKL_UNSUPPORTED
    assert lib.skl_ltlt_blk_piv(8, 0, 0, None, 8, None, 8, None, None, None, 0, None) == _capi.SKL_BAD_ARGUMENT
    assert lib.skl_apply_symmetric_pivot(4, None, 4, 2, 5, None) == _capi.SKL_BAD_PIVOT


def test_status_mapping():
    with pytest.raises(ValueError):
        _capi.check(_capi.SKL_BAD_ARGUMENT)
    with pytest.raises(InvalidVariant):
        _capi.check(_capi.SKL_UNSUPPORTED)
    with pytest.raises(IndexError):
        _capi.check(_capi.SKL_BAD_PIVOT)


def test_types_mirror_reference():
    x = SkewMatrixLower(worked_example())
    d = x.dense()
    assert np.array_equal(d, -d.T) and d[3, 2] == 5.0
    assert np.isclose(x.norm(), np.sqrt(2.0) * np.linalg.norm(np.tril(worked_example(), -1)))
    t = SkewTridiagonal(np.array([2.0, 3.0, 7.0]))
    s = form_s_splitting(t)
    sd = s.dense(float)
    assert np.array_equal(sd - sd.T, t.dense())
    assert UnitLowerFactor.identity(4).dense().tolist() == np.eye(4).tolist()
    p = PermutationVector([0, 2, 0, 0], 4)
    assert p.sign() == -1 and p.nontrivial == 1
    assert compose_permutation(p).tolist() == [0, 3, 2, 1]
    with pytest.raises(ValueError):
        PermutationVector([0, 5], 4)
    with pytest.raises(ValueError):
        SkewMatrixLower(np.zeros((3, 4)))
    e = ZeroPivot(3)
    assert e.column == 3 and isinstance(e, ArithmeticError)


def test_inputs_are_seeded_and_lower():
    a = skew_lower(50, 3)
    b = skew_lower(50, 3)
    assert np.array_equal(a, b) and a.flags.f_contiguous
    assert not np.triu(a).any()
    assert CONFIGS[2]["n"] == 4096 and CONFIGS[2]["nb"] == 128
    u = config_input(3, 0) if False else skew_lower(64, 0, "uniform")
    assert np.abs(u).max() <= 2.0


@pytest.mark.parametrize("m,b", [(5, 2), (64, 16), (129, 32), (300, 64)])
@pytest.mark.parametrize("fused", ["var1", "var2a", "var2b"])
def test_closed_form_flops_match_counted(m, b, fused):
    x = skew_lower(m, m)
    o = oracle.ltlt_blk_piv(x, b=b, fused=fused)
    assert flops_blk_piv(m, b, fused, o.pivots, o.tau) == FlopCounter(**o.flops)


@pytest.mark.parametrize("m", [2, 3, 17, 64, 101])
def test_closed_form_twostep_flops(m):
    o = oracle.ltlt_unb_twostep(skew_lower(m, m), pivot=True)
    assert flops_unb_twostep(m, o.pivots, o.tau) == FlopCounter(**o.flops)


def test_reference_schedule_shapes():
    s = reference_schedule(4096, 128, "var1")
    assert len(s) == 32 and s[0] == (0, 128, 0, 1) and s[-1][0] + s[-1][1] == 4095
    s2 = reference_schedule(1000, 100, "var2b")
    assert s2[0][1] == 101 and s2[1][2] == 100


def test_panel_view_shapes_and_block_config_roundtrip():
    import numpy as np
    from paper_2411_09859_b200.kernels2 import PanelView
    from paper_2411_09859_b200.kernels3 import get_block_config, set_block_config
    v = PanelView(np.zeros((8, 8), order="F"), 2, 5)
    assert v.square.shape == (3, 3) and v.rect.shape == (3, 3)
    saved = get_block_config()
    try:
        assert set_block_config(m_c=16, k_c=8).k_c == 8 and get_block_config().m_c == 16
    finally:
        set_block_config(m_c=saved.m_c, k_c=saved.k_c, n_c=saved.n_c)
    import paper_2411_09859_b200 as pk
    assert set(pk.LADDER) == {f"step{i}" for i in range(6)} and pk.LADDER["step0"].l2_workers == 1
