"""3D FMR golden from the REAL reference (needs /root/reference; run in the
build container, ~10 min):

    python tests/golden/make_fmr_golden.py

Runs ``magphon.sim.run`` on configs/film3d.cfg (C3's 4-cell YIG film on a Si
substrate, reduced to 32x32x16 cells, in-plane bias, weak 10 GHz drive,
83,081 steps = 0.48 ns), then ``magphon.analysis.esprit`` on the ringdown of
the film-centre magnetisation probes (after the drive pulse, decimated by
10, model order 4, 1024 Hankel columns), and ``magphon.oracle.
kittel_frequency`` for the film's bias and Ms.  Records the extracted modes,
the Kittel frequency and SHA-256 digests of every probe series, the LLG
iteration counts and the final E/H/M arrays (tests/golden/film3d_fmr.json).
It also checks that this repo's loader reads configs/film3d.cfg to the same
configuration as the reference loader.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
OUT = Path(__file__).resolve().parent / "film3d_fmr.json"
CFG = ROOT / "configs" / "film3d.cfg"

# ringdown window and ESPRIT settings (shared with tests/test_fmr3d_gpu.py)
TAIL_START, DECIMATE, ORDER, COLUMNS = 63000, 10, 4, 1024


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def modes_of(esprit, samples, dt):
    tail = np.asarray(samples)[TAIL_START::DECIMATE]
    return [{"freq": m.freq, "Q": m.Q, "amplitude": float(abs(m.amplitude)),
             "decay_rate": m.decay_rate}
            for m in esprit((tail, dt * DECIMATE), ORDER, COLUMNS)]


def main() -> None:
    from magphon import analysis, oracle
    from magphon.config import load_config as rload
    from magphon.constants import gauss_4piMs_to_si, oersted_to_si
    from magphon import sim

    from paper_2510_22221_b200.config import load_config as mload
    ref_cfg, mine = rload(str(CFG)), mload(CFG)
    assert ref_cfg.grid.cell_shape == mine.grid.cell_shape
    assert ref_cfg.grid.spacings == mine.grid.spacings and ref_cfg.t_end == mine.t_end
    assert ref_cfg.source.__dict__ == mine.source.__dict__ and ref_cfg.probes == mine.probes
    for f in ("sigma", "eps_r", "Ms", "alpha", "gamma_e", "Hbias"):
        assert np.array_equal(getattr(ref_cfg.materials, f), getattr(mine.materials, f)), f
    t0 = time.time()
    res = sim.run(ref_cfg)
    print(f"{res.steps} steps in {time.time() - t0:.0f} s", flush=True)
    dt = ref_cfg.dt
    probes = {f"{k[0]}_{k[1][0]}_{k[1][1]}_{k[1][2]}": v.samples for k, v in res.probes.items()}
    out = {
        "steps": res.steps, "dt": dt,
        "esprit": {"tail_start": TAIL_START, "decimate": DECIMATE, "order": ORDER,
                   "columns": COLUMNS},
        "modes": {name: modes_of(analysis.esprit, s, dt)
                  for name, s in probes.items() if name[0] == "M"},
        "kittel_hz": oracle.kittel_frequency(oersted_to_si(3000.0), gauss_4piMs_to_si(1750.0)),
        "probes": {name: digest(s) for name, s in probes.items()},
        "iterations": digest(np.asarray(res.iterations, dtype=np.int64)),
        "fields": {k: digest(v) for k, v in res.lattice.state_arrays().items()},
        "max_abs_probe": {name: float(np.abs(s).max()) for name, s in probes.items()},
    }
    OUT.write_text(json.dumps(out, indent=1))
    print(json.dumps(out["modes"], indent=1), out["kittel_hz"])
    print("wrote", OUT)


if __name__ == "__main__":
    main()
