"""Steady-state speed of a realistic magnetic run from rest (e.g.
configs/film3d.cfg, the 3D FMR ringdown): one handle, warm-up, then N steps
through mpb_run timed on the host; and how many steps had r* > 1."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_22221_b200 import sim  # noqa: E402
from paper_2510_22221_b200.config import load_config  # noqa: E402
from paper_2510_22221_b200.grid import initial_magnetization  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "film3d"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 2000
cfg = load_config(Path(__file__).resolve().parents[1] / "configs" / f"{name}.cfg", lazy=True)
keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in cfg.probes))
dev = sim._device_run(cfg, cfg.materials, keys, device=0)
dev.load_state(None, initial_magnetization(cfg.materials))
src = sim.source_values(cfg.source, cfg.dt, 0, warm + steps)
dev.run(0, src[:warm])
t0 = time.perf_counter()
_, iters, fail = dev.run(warm, src[warm:])
t = time.perf_counter() - t0
dev.close()
cells = int(np.prod(cfg.grid.cell_shape))
print(f"{name}: steps {warm}..{warm + steps}: {1e6 * t / steps:.2f} us/step = "
      f"{cells * steps / t / 1e9:.3f} Gcell/s; r* histogram {np.bincount(iters).tolist()}, "
      f"failure {fail}")
