"""CPU baselines per BASELINE config (SURVEY 8d "CPU baseline timing"): the
numpy oracle (restatement of the reference, single-threaded like its numpy
ufuncs) for K steps of each config, plus the all-cores replica aggregate
(the reference's own sweep parallelism) for C1 and C2.  Runs on the GPU box's
host; prints one JSON line per measurement.

    python tools/cpu_configs.py
"""
import json
import os
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from oracle import magphon_oracle as orc  # noqa: E402
from paper_2510_22221_b200.config import load_config  # noqa: E402

STEPS = {"c1": 300, "c2": 50, "c3": 20, "c4": 3}


def main():
    for name, steps in STEPS.items():
        cfg = load_config(ROOT / "configs" / f"{name}.cfg", lazy=False)
        cells = int(np.prod(cfg.grid.cell_shape))
        cfg = replace(cfg, t_end=(steps + 0.5) * cfg.dt)
        orc.run(cfg, n_steps=1)
        t0 = time.perf_counter()
        orc.run(cfg, n_steps=steps)
        dt = time.perf_counter() - t0
        print(json.dumps({"config": name, "cells": cells, "steps": steps, "cores": 1,
                          "seconds": dt, "gcell_updates_per_s": cells * steps / dt / 1e9}),
              flush=True)
    for name in ("c1", "c2"):
        procs = bench.host_cores_for_replicas(name)
        steps = 20 if name == "c2" else 100
        bench.cpu_replicas(name, 1, procs)
        v, secs, cells = bench.cpu_replicas(name, steps, procs)
        print(json.dumps({"config": name, "cells": cells, "steps": steps, "cores": procs,
                          "mode": "replicas", "seconds": secs, "gcell_updates_per_s": v}),
              flush=True)


if __name__ == "__main__":
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    main()
