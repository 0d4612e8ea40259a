"""Driver calls whose reference CallTrace is pinned in traces.json (make_traces.py).
Each case: (key, kind, kwargs); inputs are skew_lower(n, seed)."""

TRACE_CASES = []
for fused, n in (("var1", 64), ("var2a", 64), ("var2b", 65), ("var1", 300)):
    TRACE_CASES.append((f"piv_{fused}_{n}", "blk_piv", dict(n=n, seed=3, b=16, fused=fused)))
for driver in ("var1", "var2a", "var2b", "twostep", "left"):
    for pv in ("ll", "rl", "twostep"):
        TRACE_CASES.append((f"blk_{driver}_{pv}", "blk", dict(n=48, seed=4, b=8, driver=driver, pv=pv)))
for pivot in (False, True):
    TRACE_CASES.append((f"unb_twostep_{pivot}", "unb_twostep", dict(n=40, seed=5, pivot=pivot)))
    TRACE_CASES.append((f"unb_ll_{pivot}", "unb_ll", dict(n=40, seed=6, pivot=pivot)))
    TRACE_CASES.append((f"unb_rl_{pivot}", "unb_rl", dict(n=40, seed=7, pivot=pivot)))
TRACE_CASES.append(("unb_ll_fc", "unb_ll", dict(n=30, seed=8, pivot=False, first_column=True)))
for pv in ("ll", "rl", "twostep"):
    TRACE_CASES.append((f"unb_panel_{pv}", "unb_panel", dict(n=40, seed=9, width=10, variant=pv, pivot=False)))
TRACE_CASES.append(("unb_panel_piv", "unb_panel", dict(n=40, seed=9, width=10, variant="ll", pivot=True)))


def first_column_vec(n):
    import numpy as np
    return np.linspace(-1.0, 1.0, n - 1)


def run_case(mod, kind, kw, skew_lower):
    """Call the driver of ``mod`` (the reference package or ours) for one case."""
    x = mod.SkewMatrixLower(skew_lower(kw["n"], kw["seed"]))
    if kind == "blk_piv":
        return mod.ltlt_blk_piv(x, b=kw["b"], fused=kw["fused"])
    if kind == "blk":
        return getattr(mod, f"ltlt_blk_{kw['driver']}")(x, b=kw["b"], panel_variant=kw["pv"])
    if kind == "unb_twostep":
        return mod.ltlt_unb_twostep(x, pivot=kw["pivot"])
    if kind == "unb_ll":
        fc = first_column_vec(kw["n"]) if kw.get("first_column") else None
        return mod.ltlt_unb_ll(x, pivot=kw["pivot"], first_column=fc)
    if kind == "unb_rl":
        return mod.ltlt_unb_rl(x, pivot=kw["pivot"])
    if kind == "unb_panel":
        return mod.ltlt_unb_panel(x, kw["width"], variant=kw["variant"], pivot=kw["pivot"])
    raise ValueError(kind)
