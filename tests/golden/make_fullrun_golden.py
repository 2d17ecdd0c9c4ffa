"""Full-length golden of the reference's only shipped run, from the REAL
reference (needs /root/reference; run in the build container):

    python tests/golden/make_fullrun_golden.py

Runs ``magphon.sim.run`` on ``pkg/configs/cavity1d.cfg`` for its full 3 ns
(499,655 steps) and records SHA-256 digests of the probe series, the LLG
iteration counts and the final E/H/M arrays (the raw data is ~8 MB), plus a
few summary numbers.  It also checks that this repo's ``configs/cavity1d.cfg``
loads, with the reference loader, to the same configuration as the shipped
file.  Output: tests/golden/cavity1d_full.json.
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
OUT = Path(__file__).resolve().parent / "cavity1d_full.json"


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def main() -> None:
    from magphon import config, sim
    shipped = config.load_config("/root/reference/pkg/configs/cavity1d.cfg")
    ours = config.load_config(str(ROOT / "configs" / "cavity1d.cfg"))
    for f in ("cfl_factor", "t_end", "probes", "bias_sweep", "bias_direction",
              "spectrum_probe", "llg_params", "boundaries", "source"):
        assert getattr(shipped, f) == getattr(ours, f), f
    assert shipped.grid == ours.grid
    for f in ("sigma", "eps_r", "Ms", "alpha", "gamma_e", "Hbias"):
        assert np.array_equal(getattr(shipped.materials, f), getattr(ours.materials, f)), f
    t0 = time.time()
    res = sim.run(shipped)
    print(f"{res.steps} steps in {time.time() - t0:.0f} s", flush=True)
    out = {"steps": res.steps,
           "probes": {f"{k[0]}_{k[1][0]}_{k[1][1]}_{k[1][2]}": digest(v.samples)
                      for k, v in res.probes.items()},
           "iterations": digest(np.asarray(res.iterations, dtype=np.int64)),
           "fields": {k: digest(v) for k, v in res.lattice.state_arrays().items()},
           "r_star_counts": {str(int(r)): int(c) for r, c in
                             zip(*np.unique(res.iterations, return_counts=True))},
           "max_abs_probe": {f"{k[0]}_{k[1][0]}_{k[1][1]}_{k[1][2]}":
                             float(np.abs(v.samples).max()) for k, v in res.probes.items()}}
    OUT.write_text(json.dumps(out, indent=1))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
