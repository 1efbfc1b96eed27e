"""Small shared test helpers (no method arithmetic)."""


def copy_sd(sd, **over):
    """A subdomain-like object with copied arrays and some fields overridden."""
    d = dict(n=sd.n, m=sd.m, L_colptr=sd.L_colptr.copy(), L_rowidx=sd.L_rowidx.copy(), perm=sd.perm.copy(),
             Bt_colptr=sd.Bt_colptr.copy(), Bt_rowidx=sd.Bt_rowidx.copy(), Bt_values=sd.Bt_values.copy(),
             lambda_map=sd.lambda_map.copy())
    d.update(over)
    return type("SD", (), d)
