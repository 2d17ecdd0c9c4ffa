"""Fraction of lattice entries holding tiny values (0 < |x| < 2^-969, the
exact-division guard's range: such a curl batch takes the out-of-line IEEE
path) in a run from rest, after N steps."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_22221_b200 import sim  # noqa: E402
from paper_2510_22221_b200.config import load_config  # noqa: E402
from paper_2510_22221_b200.grid import initial_magnetization  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
init = "zero"
if name.endswith(":random"):
    name, init = name.split(":")[0], "random"
cfg = load_config(Path(__file__).resolve().parents[1] / "configs" / f"{name}.cfg", lazy=True)
dev = sim._device_run(cfg, cfg.materials, [], device=0)
if init == "random":
    import bench
    dev.load_state(bench.synthetic_state(cfg.grid.field_shape, "random"),
                   initial_magnetization(cfg.materials))
else:
    dev.load_state(None, initial_magnetization(cfg.materials))
done = 0
for n in [int(x) for x in sys.argv[2:]] or [100, 300, 600, 1200]:
    dev.run(done, sim.source_values(cfg.source, cfg.dt, done, n))
    done = n
    st = dev.save_state()
    tiny = 2.0 ** -969
    parts = []
    for k in ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz"):
        a = np.abs(st[k])
        parts.append(f"{k} zero {np.mean(a == 0):.3f} tiny {np.mean((a > 0) & (a < tiny)):.3f} "
                     f"subn {np.mean((a > 0) & (a < 2.2250738585072014e-308)):.3f}")
    print(f"step {n}: " + " | ".join(parts), flush=True)
dev.close()
