"""Diagnostic: first step / plane where the emulated slab run departs from
the single-domain run."""
import sys
from dataclasses import replace

import numpy as np

sys.path.insert(0, ".")
from paper_2510_22221_b200 import parallel, sim  # noqa: E402
from tests.golden.cases import CASES, build, mirror_namespace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "mixed3d"
nr = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg0 = build(CASES[name], mirror_namespace())
print("slabs", [(s.x_lo, s.x_hi, s.field_range, s.cell_range) for s in parallel.make_slabs(cfg0.grid.nx, nr)])
for k in [int(a) for a in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["1","2","3","5","10"])]:
    cfg = replace(cfg0, t_end=(k - 0.5) * cfg0.dt)
    ref = sim.run(cfg)
    f, M, pr, its = parallel.run_group(cfg, nr)
    bad = []
    for n, v in ref.lattice.state_arrays().items():
        got = M if n == "M" else f[n]
        if not np.array_equal(got, v):
            d = np.abs(got - v)
            planes = sorted(set(np.nonzero(d)[1 if n == "M" else 0].tolist()))
            bad.append((n, float(d.max()), planes[:10]))
    di = [i for i, (a, b) in enumerate(zip(its.tolist(), ref.iterations.tolist())) if a != b]
    print("steps", k, "iter mismatch at", di[:5], "bad", bad)
    if bad:
        break
