"""Bias-sweep throughput on one GPU (BASELINE configs[1]: C2 swept through
the anti-crossing): serial runs vs several concurrent runs per GPU.

    python tools/sweep_throughput.py [--config c2] [--biases 8] [--steps 400]

Prints one JSON line per concurrency level (aggregate Gcell-updates/s over the
whole sweep, wall clock around sim.sweep, FFT post-processing included).
"""
import argparse
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2510_22221_b200 import sim  # noqa: E402
from paper_2510_22221_b200.config import load_config  # noqa: E402
from paper_2510_22221_b200.constants import oersted_to_si  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--biases", type=int, default=8)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--levels", default="1,2,4,8")
    a = ap.parse_args()
    cfg = load_config(ROOT / "configs" / f"{a.config}.cfg")
    cfg = replace(cfg, t_end=(a.steps - 0.5) * cfg.dt)
    biases = [oersted_to_si(b) for b in np.linspace(1500.0, 2100.0, a.biases)]
    cells = int(np.prod(cfg.grid.cell_shape))
    sim.sweep(cfg, biases=biases[:1])                      # warm-up (context, allocator)
    ref = None
    for k in (int(x) for x in a.levels.split(",")):
        t0 = time.perf_counter()
        smap = sim.sweep(cfg, biases=biases, parallel=k)
        t = time.perf_counter() - t0
        if ref is None:
            ref = smap.mags
        same = bool(np.array_equal(ref, smap.mags))
        print(json.dumps({"config": a.config, "biases": a.biases, "steps": a.steps,
                          "concurrent_per_gpu": k, "seconds": t,
                          "gcell_updates_per_s": cells * a.steps * a.biases / t / 1e9,
                          "identical_to_serial": same}), flush=True)


if __name__ == "__main__":
    main()
