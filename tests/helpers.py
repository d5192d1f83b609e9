"""Shared test helpers: run the same seeded inputs through the oracle and libmem and compare.

Tolerances (north_star): integer/index layers bit-exact; fp32 layers
|gpu - oracle| <= 1e-6 + 1e-5 |oracle| with NaN == NaN.
"""
import numpy as np

ATOL, RTOL = 1e-6, 1e-5

INT_SUFFIXES = ("valid", "_observed", "_label")


def is_int_layer(name):
    return name == "valid" or name.endswith("_observed") or name.endswith("_label")


def compare_layers(gpu_map, ora_map, names=None, where="", exact=True):
    """returns dict name -> max abs diff; asserts the parity bar.  With exact=True (the
    default) every layer must also equal the oracle BIT FOR BIT: every point path sums in the
    oracle's order or in certified-exact arithmetic (reading D39), and the image
    path evaluates the oracle's expressions in its order."""
    names = names or gpu_map.layer_names()
    out = {}
    for nm in names:
        g = np.asarray(gpu_map.get_layer(nm))
        o = ora_map.get_layer(nm)
        assert g.shape == o.shape, (nm, g.shape, o.shape)
        nan_g, nan_o = np.isnan(g), np.isnan(o)
        assert (nan_g == nan_o).all(), f"{where}{nm}: NaN pattern differs at {np.argwhere(nan_g != nan_o)[:5]}"
        if is_int_layer(nm):
            bad = g != o
            assert not bad.any(), f"{where}{nm}: {bad.sum()} integer mismatches, first {np.argwhere(bad)[:5]}"
            out[nm] = 0.0
        else:
            gg, oo = g[~nan_g].astype(np.float64), o[~nan_o].astype(np.float64)
            d = np.abs(gg - oo)
            tol = ATOL + RTOL * np.abs(oo)
            bad = d > tol
            assert not bad.any(), f"{where}{nm}: {bad.sum()} values beyond tolerance, max diff {d.max()}"
            if exact:
                neq = gg != oo
                assert not neq.any(), f"{where}{nm}: {neq.sum()} values differ from the oracle in the last bits (max {d.max()})"
            out[nm] = float(d.max()) if d.size else 0.0
    return out


def copy_state_to_oracle(gpu_map, ora_map):
    """single-step parity: the oracle takes the GPU's stored state."""
    for nm in gpu_map.layer_names():
        v = np.asarray(gpu_map.get_layer(nm))
        try:
            ora_map.set_layer(nm, v)
        except Exception:
            pass  # derived layers (class_bayesian theta) are read-only on both sides


def noise_dict(n):
    return dict(n)
