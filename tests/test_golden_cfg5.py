"""CPU checks of the config-5 golden (one run of the unmodified reference at
n=49152, nb=512; tests/golden/make_cfg5.py): the fixture is self-consistent, and
the host replay of the reference's flop accounting (instrument.flops_blk_piv,
instrument.py:14-40 rules) reproduces the reference's own tallies from the
fixture's pivots and tau -- the accounting is pinned at the largest config too."""
import numpy as np

import oracle
from paper_2411_09859_b200.instrument import flops_blk_piv


def test_cfg5_golden_consistent(golden):
    g = golden("cfg5_n49152_b512.npz")
    n = int(g["n"])
    piv = g["piv"].astype(np.int64)
    tau = g["tau"]
    assert n == 49152 and int(g["b"]) == 512
    assert piv.shape == (n,) and tau.shape == (n - 1,)
    assert piv[0] == 0 and piv[-1] == 0
    assert np.all(piv >= 0) and np.all(piv + np.arange(n) < n)
    sign, lg = oracle.pfaffian_slog(tau, piv, n)
    assert sign == float(g["sign"]) and abs(lg - float(g["logpf"])) <= 1e-12 * abs(lg)
    assert np.all(np.isfinite(g["lr"])) and np.all(np.isfinite(g["ltr"]))


def test_cfg5_flop_replay_matches_reference(golden):
    g = golden("cfg5_n49152_b512.npz")
    fc = flops_blk_piv(int(g["n"]), int(g["b"]), "var1", g["piv"].astype(np.int64), g["tau"])
    assert [fc.level2, fc.level3, fc.panel, fc.pivot] == [int(v) for v in g["flops"]]
