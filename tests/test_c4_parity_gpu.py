"""The headline benchmark configuration itself (C4, 1024x1024x128 cells,
BASELINE configs[3]) on the CUDA path vs the CPU oracle, bit for bit.

bench.py times C4 from a synthetic mid-run state; here the same grid resumes
from a mid-run state (random E/H on every physical entry, M tilted off the
bias so the LLG fixed point takes several iterates) and takes 3 coupled
steps through ``sim.run`` -- the public entry point -- on the GPU and in the
numpy oracle (a restatement of magphon.sim.run pinned to the reference's own
goldens).  Every field array, M, every probe sample and r* per step must be
identical (np.array_equal).  The sweep runs in the tile form bench.py times
(two 256-thread CTAs per SM, 512-entry tiles, 8 x-chunks of 128 planes),
which the test pins through mpb_sweep_form.

Host memory: ~70 GB (the oracle's dense per-cell arrays and temporaries);
~50 s of single-core oracle time.
"""
from dataclasses import replace
from pathlib import Path

import numpy as np
import pytest

from oracle import magphon_oracle as orc
from paper_2510_22221_b200 import sim
from paper_2510_22221_b200.config import load_config
from tests.test_configs_gpu import mid_run_state

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _enough_host_memory(gb):
    try:
        import psutil
        return psutil.virtual_memory().available > gb * (1 << 30)
    except ImportError:
        return True


@pytest.mark.skipif(not _enough_host_memory(90), reason="needs ~90 GB of host RAM")
def test_c4_three_steps_match_oracle_bitwise():
    cfg = load_config(ROOT / "configs" / "c4.cfg")
    start, steps = 200, 3
    cfg = replace(cfg, t_end=(start + steps - 0.5) * cfg.dt)
    assert cfg.n_steps == start + steps
    keys = [(p[0], (p[1], p[2], p[3])) for p in cfg.probes]
    state = mid_run_state(cfg, 11)
    snap = {"fields": state, "step": start, "probes": {k: np.zeros(start) for k in keys},
            "iterations": np.ones(start, dtype=int)}
    # the tile form bench.py times on this grid
    dev = sim._device_run(load_config(ROOT / "configs" / "c4.cfg", lazy=True),
                          load_config(ROOT / "configs" / "c4.cfg", lazy=True).materials, keys)
    try:
        form = dev.sweep_form()
    finally:
        dev.close()
    assert form == {"V": 2, "NT": 256, "T": 512, "chunks": 8}, form
    res = sim.run(cfg, resume=snap)             # loads (copies) the state, GPU steps
    got = res.lattice.state_arrays()
    ref = orc.run(cfg, resume=snap)             # the oracle works on its own copy
    assert res.steps == ref["steps"] == start + steps
    for k, v in ref["fields"].items():
        same = np.array_equal(got[k], v)
        assert same, (k, float(np.max(np.abs(got[k] - v))))
    assert np.array_equal(res.iterations, ref["iterations"])
    assert int(np.max(ref["iterations"][start:])) >= 2        # non-trivial fixed point
    for key, v in ref["probes"].items():
        assert np.array_equal(res.probes[key].samples, v), key
