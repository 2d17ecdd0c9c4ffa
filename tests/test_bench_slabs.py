"""bench.py's multi-GPU set-up (slab_run) on the CPU: the per-rank grid,
painted slab materials and state shapes for weak (C4 repeated along x) and
strong (C5 split) scaling.  DeviceRun is replaced by a recorder -- the device
side of slabs is covered by tests/test_slab_gpu.py."""
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2510_22221_b200 import engine, parallel  # noqa: E402
from paper_2510_22221_b200.config import load_config  # noqa: E402


class Recorder:
    last = None

    def __init__(self, grid, mats, boundaries, src_loc, src_pol, keys, llg, dt, device=0,
                 kernel_variant=0, slab=None):
        ids, table = engine.material_table(mats, dt, grid.spacings)
        Recorder.last = self
        self.grid, self.mats, self.keys, self.slab, self.ids = grid, mats, keys, slab, ids
        self.src_loc = src_loc
        self.probes = keys

    def load_state(self, fields, M):
        self.fields, self.M = fields, M


class Args:
    variant = 0
    init = "zero"


@pytest.mark.parametrize("name,scaling,world", [("c2", "weak", 4), ("c3", "strong", 3)])
def test_slab_run_layout(name, scaling, world, monkeypatch):
    monkeypatch.setattr(engine, "DeviceRun", Recorder)
    monkeypatch.setattr(parallel, "nccl_unique_id", lambda dist: bytes(range(128)))
    cfg = load_config(ROOT / "configs" / f"{name}.cfg")
    keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in cfg.probes))
    args = Args()
    args.scaling = scaling
    g = cfg.grid
    gnx = g.nx * world if scaling == "weak" else g.nx
    owned = 0
    for rank in range(world):
        dev, cells = bench.slab_run(cfg, keys, world, rank, 0, args)
        r = Recorder.last
        sl = r.slab
        assert r.grid.cell_shape == (gnx, g.ny, g.nz)
        assert sl.rank == rank and sl.nranks == world and sl.nccl_id == bytes(range(128))
        c0, c1 = sl.cell_range
        f0, f1 = sl.field_range
        assert r.mats.shape == (c1 - c0, g.ny, g.nz) and r.ids.shape == r.mats.shape
        assert r.fields["Ex"].shape == (f1 - f0, g.ny + 1, g.nz + 1)
        assert r.M.shape == (3, c1 - c0, g.ny, g.nz)
        assert cells == (sl.x_hi - sl.x_lo) * g.ny * g.nz
        assert (r.keys == []) == (scaling == "weak")
        owned += sl.x_hi - sl.x_lo
        # the slab's materials are the config's (periodically, for weak scaling)
        dense = load_config(ROOT / "configs" / f"{name}.cfg", lazy=False).materials
        period = np.arange(c0, c1) % g.nx
        assert np.array_equal(np.asarray(r.mats.Ms), np.asarray(dense.Ms)[period])
    assert owned == gnx
