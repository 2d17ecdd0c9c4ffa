"""Run-to-run determinism at benchmark size: the same mid-run state stepped
twice must give the same bits.  The CUDA path has no atomics on field values
and one writer per entry, so any race (the single-barrier ring, bulk stores,
the overlapped slab exchange) would show up here as a mismatch."""
import hashlib
from pathlib import Path

import numpy as np
import pytest

from paper_2510_22221_b200 import sim
from paper_2510_22221_b200.config import load_config
from paper_2510_22221_b200.grid import initial_magnetization

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _digest_run(cfg, state, start, steps):
    keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in cfg.probes))
    dev = sim._device_run(cfg, cfg.materials, keys)
    try:
        dev.load_state({k: state[k] for k in ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")}, state["M"])
        probes, iters, fail = dev.run(start, sim.source_values(cfg.source, cfg.dt, start,
                                                               start + steps))
        assert fail is None
        out = dev.save_state()
    finally:
        dev.close()
    h = hashlib.sha256()
    for k in sorted(out):
        h.update(np.ascontiguousarray(out[k]).tobytes())
    h.update(probes.tobytes())
    h.update(iters.tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name,steps", [("c3", 60), ("c4", 40)])
def test_benchmark_size_runs_are_deterministic(name, steps):
    cfg = load_config(ROOT / "configs" / f"{name}.cfg")
    rng = np.random.default_rng(17)
    fs = cfg.grid.field_shape
    state = {}
    for q, k in enumerate(("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")):
        a = rng.standard_normal(fs)
        a *= 1e3 if k[0] == "E" else 2.65
        state[k] = a
    state["M"] = initial_magnetization(cfg.materials)
    a = _digest_run(cfg, state, 100, steps)
    b = _digest_run(cfg, state, 100, steps)
    assert a == b


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_graph_and_eager_launch_counts_agree(name):
    """The launch count reported for CUDA-graph replays (bench `gpu_launches`,
    e2e leg) is the number of kernels captured, i.e. the eager count."""
    cfg = load_config(ROOT / "configs" / f"{name}.cfg")
    keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in cfg.probes))
    counts = []
    for timed in (True, False):          # timed: eager launches; else graphs
        dev = sim._device_run(cfg, cfg.materials, keys)
        try:
            fs = cfg.grid.field_shape
            dev.load_state({k: np.zeros(fs) for k in ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")},
                           initial_magnetization(cfg.materials))
            dev.set_kernel_timing(timed)
            _, _, fail = dev.run(0, sim.source_values(cfg.source, cfg.dt, 0, 32))
            assert fail is None
            counts.append(dev.launch_count())
        finally:
            dev.close()
    assert counts[0] == counts[1] > 0, counts
