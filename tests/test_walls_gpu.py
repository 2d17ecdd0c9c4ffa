"""Every x/y wall combination on the CUDA path vs the CPU oracle, bit for bit.

The x0, x1, y0, y1 walls run as ONE launch (k_walls_xy) that must reproduce
the reference's sequential face order (em.py:324-359) on the edge lines where
the faces interact: a y wall overwrites Ez on the x walls' rows, and a y
wall's MUR1 reads Ez on its inner row after an x wall wrote it.  All 81
combinations of PEC / PMC / MUR1 on those four faces (z walls MUR1 / PEC),
from a random mid-run state so every wall entry is nonzero, on the fused
launch and on the one-launch-per-face form (MPB_WALLS=face).
"""
import itertools

import numpy as np
import pytest

from oracle import magphon_oracle as orc
from paper_2510_22221_b200 import em, sim
from paper_2510_22221_b200.constants import oersted_to_si
from paper_2510_22221_b200.grid import GridSpec
from paper_2510_22221_b200.materials import MaterialCell, MaterialMap
from tests.test_configs_gpu import mid_run_state

pytestmark = pytest.mark.gpu

KINDS = ("PEC", "PMC", "MUR1")
STEPS = 3
START = 10


def _config(x0, x1, y0, y1):
    grid = GridSpec(7, 6, 5, 4e-6, 5e-6, 3e-6)
    mm = MaterialMap(grid.cell_shape, MaterialCell(sigma=0.0, eps_r=2.0))
    mm.fill_box(MaterialCell(eps_r=9.0), 0, 7, 0, 1, 0, 5)          # a y0-side layer
    mm.fill_box(MaterialCell(eps_r=15.0, Ms=9.7e5, alpha=0.01,
                             Hbias=(oersted_to_si(1500.0), 0.0, 0.0)), 0, 2, 4, 6, 1, 4)
    mm.freeze()
    dt = em.cfl_timestep(grid, 0.9)
    return sim.SimConfig(
        grid=grid, materials=mm,
        source=em.SourceSpec(f0=80e9, Tp=1e-12, amplitude=1e3, location=(3, 3, 2),
                             polarization=(0.0, 0.0, 1.0)),
        boundaries=em.BoundarySpec(x0=x0, x1=x1, y0=y0, y1=y1, z0="MUR1", z1="PEC"),
        cfl_factor=0.9, t_end=(START + STEPS - 0.5) * dt,
        probes=(("Ez", 0, 0, 2), ("Ez", 7, 6, 2), ("Ey", 0, 3, 1), ("Ex", 3, 0, 1)))


@pytest.mark.parametrize("per_face", [False, True])
def test_all_xy_wall_combinations_match_oracle(per_face, monkeypatch):
    if per_face:
        monkeypatch.setenv("MPB_WALLS", "face")
    bad = []
    for x0, x1, y0, y1 in itertools.product(KINDS, repeat=4):
        cfg = _config(x0, x1, y0, y1)
        keys = [(p[0], (p[1], p[2], p[3])) for p in cfg.probes]
        snap = {"fields": mid_run_state(cfg, 11), "step": START,
                "probes": {k: np.zeros(START) for k in keys},
                "iterations": np.ones(START, dtype=int)}
        ref = orc.run(cfg, resume={**snap, "fields": {k: v.copy()
                                                      for k, v in snap["fields"].items()}})
        res = sim.run(cfg, resume=snap)
        got = res.lattice.state_arrays()
        for k, v in ref["fields"].items():
            if not np.array_equal(got[k], v):
                bad.append((x0, x1, y0, y1, k))
        for key, v in ref["probes"].items():
            if not np.array_equal(res.probes[key].samples, v):
                bad.append((x0, x1, y0, y1, key))
    assert not bad, bad[:10]
