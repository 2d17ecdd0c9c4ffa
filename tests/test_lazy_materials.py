"""Lazy (painted) material maps give the device exactly what dense maps do.

The lazy path exists for grids whose dense per-cell arrays do not fit in host
memory (C5); these checks run on the CPU at sizes where both paths fit.
"""
from pathlib import Path

import numpy as np
import pytest

from paper_2510_22221_b200 import engine
from paper_2510_22221_b200.config import load_config
from paper_2510_22221_b200.grid import initial_magnetization
from paper_2510_22221_b200.parallel import _MaterialSlab, make_slabs
from paper_2510_22221_b200.sim import _materials_with_bias

ROOT = Path(__file__).resolve().parents[1]
FIELDS = ("ca", "cb", "Ms", "alpha_ms", "c_llg", "magnetic", "eps")


def per_cell(materials, dt, spacings):
    ids, table = engine.material_table(materials, dt, spacings)
    out = {}
    for f in FIELDS:
        col = np.array([getattr(table[q], f) for q in range(len(table))])
        out[f] = col[ids]
    for a in range(3):
        out[f"mur_k{a}"] = np.array([table[q].mur_k[a] for q in range(len(table))])[ids]
        out[f"hbias{a}"] = np.array([table[q].hbias[a] for q in range(len(table))])[ids]
    return out


def same(a, b):
    return np.array_equal(a.view(np.int64), b.view(np.int64)) if a.dtype == np.float64 \
        else np.array_equal(a, b)


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_lazy_map_matches_dense(name):
    dense = load_config(ROOT / "configs" / f"{name}.cfg", lazy=False)
    lazy = load_config(ROOT / "configs" / f"{name}.cfg", lazy=True)
    assert lazy.materials.lazy and not lazy.materials.dense
    g = dense.grid
    sp = (g.dx, g.dy, g.dz)
    pd, pl = per_cell(dense.materials, dense.dt, sp), per_cell(lazy.materials, dense.dt, sp)
    mag = np.asarray(dense.materials.Ms) > 0
    for f in pd:
        if f.startswith("hbias"):          # only meaningful in magnetic cells
            assert same(pd[f][mag], pl[f][mag]), f
        else:
            assert same(pd[f], pl[f]), f
    assert same(initial_magnetization(dense.materials), initial_magnetization(lazy.materials))
    assert lazy.materials.magnetic_count() == int(np.count_nonzero(mag))
    assert not lazy.materials.dense          # nothing above materialised it
    # reading a dense array materialises it, identical to the eager map
    for f in ("sigma", "eps_r", "Ms", "alpha", "gamma_e", "Hbias"):
        assert same(np.asarray(getattr(lazy.materials, f)), np.asarray(getattr(dense.materials, f)))


def test_lazy_region_and_bias_override():
    dense = load_config(ROOT / "configs" / "c3.cfg", lazy=False)
    lazy = load_config(ROOT / "configs" / "c3.cfg", lazy=True)
    g = dense.grid
    sp = (g.dx, g.dy, g.dz)
    for sl in make_slabs(g.nx, 3, True):
        d = _MaterialSlab(dense.materials, sl)
        z = _MaterialSlab(lazy.materials, sl)
        assert z.lazy and z.shape == d.shape
        pd, pl = per_cell(d, dense.dt, sp), per_cell(z, dense.dt, sp)
        for f in ("ca", "cb", "Ms", "alpha_ms", "magnetic"):
            assert same(pd[f], pl[f]), f
        assert same(initial_magnetization(d), initial_magnetization(z))
    bd = _materials_with_bias(dense.materials, 2.5e4, (0.0, 1.0, 1.0))
    bl = _materials_with_bias(lazy.materials, 2.5e4, (0.0, 1.0, 1.0))
    assert bl.lazy
    assert same(initial_magnetization(bd), initial_magnetization(bl))


@pytest.mark.parametrize("c0,c1", [(0, 65), (63, 130), (127, 257), (1, 2), (200, 600)])
def test_tiled_region_is_periodic_slice(c0, c1):
    """Weak-scaling slabs (bench.py): the config repeated along x."""
    dense = load_config(ROOT / "configs" / "c2.cfg", lazy=False)
    lazy = load_config(ROOT / "configs" / "c2.cfg", lazy=True)
    nx = dense.grid.nx
    period = np.arange(c0, c1) % nx
    t = lazy.materials.tiled_region(c0, c1)
    assert t.shape == (c1 - c0,) + dense.materials.shape[1:]
    for f in ("sigma", "eps_r", "Ms", "alpha", "gamma_e"):
        assert same(np.asarray(getattr(t, f)), np.asarray(getattr(dense.materials, f))[period]), f
    assert same(np.asarray(t.Hbias), np.asarray(dense.materials.Hbias)[:, period])
