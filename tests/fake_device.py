"""A DeviceRun stand-in for CPU tests of bench.py's multi-rank set-up
(selected with MPB_BENCH_DEVICE=tests.fake_device:Recorder): it records the
arguments and builds the material table the real engine would, but owns no
device state."""
from paper_2510_22221_b200 import engine


class Recorder:
    def __init__(self, grid, mats, boundaries, src_loc, src_pol, keys, llg, dt, device=0,
                 kernel_variant=0, slab=None):
        self.ids, self.table = engine.material_table(mats, dt, grid.spacings)
        self.grid, self.mats, self.keys, self.slab = grid, mats, keys, slab
        self.src_loc = src_loc
        self.probes = keys

    def load_state(self, fields, M):
        self.fields, self.M = fields, M
