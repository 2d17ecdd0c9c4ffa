"""Golden values for the anti-crossing acceptance test (GPU side:
tests/test_acceptance_gpu.py), generated from the REAL reference.

Run in the build container (needs /root/reference; the GPU box does not):

    python tests/golden/make_acceptance_golden.py

The reference's acceptance suite (pkg/tests/test_acceptance.py:25-240) drives
a 1D PMC cavity (nz = 917, dz = 4 um, one YIG cell in the middle) through a
bias sweep and checks the ESPRIT ringdown modes against its layered analytic
model.  This script records, per bias of that sweep:

* the analytic absorption peaks (reference magphon.oracle.CavityModel1D /
  absorbed_power on the reference's 70001-point grid + scipy find_peaks);
* the ESPRIT modes the reference itself extracts from its own FDTD run
  (magphon.sim.run + magphon.analysis.esprit, same windowing as the suite);

plus the bare-cavity mode, the drive-amplitude sweep at 1700 Oe and the Kittel
crossing bias.  Output: tests/golden/acceptance.json.
"""

from __future__ import annotations

import json
import math
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

OUT = Path(__file__).resolve().parent / "acceptance.json"

NZ, DZ = 917, 4e-6
MAG = (NZ - 1) // 2
SIGMA_C = 1.2520467594271872e-4
EPS_C = 8.168870103908924
MS = 9.7e5
ALPHA = 0.003
BIASES_OE = (500.0, 1705.3, 1780.3, 1855.3, 1930.3, 2005.3)
AMPLITUDES = (1e3, 1e4, 1e5, 1e6)


def main() -> None:
    from scipy.signal import find_peaks

    from magphon import analysis, em, oracle, sim
    from magphon.constants import CONSTANTS, oersted_to_si
    from magphon.grid import GridSpec
    from magphon.materials import MaterialCell, MaterialMap

    def config(bias_oe, amplitude=1e3, magnet=True):
        grid = GridSpec(1, 1, NZ, DZ, DZ, DZ)
        mm = MaterialMap(grid.cell_shape, MaterialCell(sigma=SIGMA_C, eps_r=EPS_C))
        if magnet:
            mm.fill_box(MaterialCell(sigma=1e-3, eps_r=1.0, Ms=MS, alpha=ALPHA,
                                     Hbias=(oersted_to_si(bias_oe), 0.0, 0.0)),
                        0, 1, 0, 1, MAG, MAG + 1)
        mm.freeze()
        return sim.SimConfig(
            grid=grid, materials=mm,
            source=em.SourceSpec(f0=14.3e9, Tp=50e-12, amplitude=amplitude,
                                 location=(0, 0, 25), polarization=(1, 0, 0)),
            boundaries=em.BoundarySpec(z0="PMC", z1="PMC"), cfl_factor=0.9,
            t_end=1.2e-9, probes=(("Ex", 0, 0, 150), ("Mz", 0, 0, MAG)))

    def modes_of(res):
        p = res.probes[("Ex", (0, 0, 150))]
        tail = p.samples[30000:]
        ms = analysis.esprit((tail[::5], p.dt_sample * 5), 6, 1024)
        drive = max(np.abs(p.samples).max(), 1.0)
        return [{"freq": m.freq, "amplitude": abs(m.amplitude)} for m in ms
                if 10e9 < m.freq < 18e9 and abs(m.amplitude) > 1e-7 * drive]

    d3 = NZ * DZ
    model = oracle.CavityModel1D(d1=d3 / 2 - DZ / 2, d2=d3 / 2 + DZ / 2, d3=d3,
                                 sigma_m=1e-3, sigma_c=SIGMA_C, eps_m=1.0, eps_c=EPS_C,
                                 Ms=MS, gamma=CONSTANTS.gamma_eff, alpha=ALPHA)
    out = {"biases_oe": list(BIASES_OE), "amplitudes": list(AMPLITUDES), "sweep": {},
           "analytic_peaks": {}, "amplitude_sweep": {}}
    freqs = np.linspace(11e9, 18e9, 70001)
    for b in BIASES_OE:
        t0 = time.time()
        P = np.array([oracle.absorbed_power(model, 2 * math.pi * f, oersted_to_si(b))
                      for f in freqs])
        pk, _ = find_peaks(P, height=P.max() * 0.005)
        out["analytic_peaks"][str(b)] = [float(f) for f in freqs[pk]]
        out["sweep"][str(b)] = modes_of(sim.run(config(b)))
        print(f"bias {b}: analytic {out['analytic_peaks'][str(b)]}, "
              f"{len(out['sweep'][str(b)])} modes ({time.time() - t0:.0f} s)", flush=True)
    out["bare_cavity"] = modes_of(sim.run(config(0.0, magnet=False)))
    for a in AMPLITUDES:
        out["amplitude_sweep"][str(a)] = modes_of(sim.run(config(1700.0, amplitude=a)))
    out["crossing_bias_oe"] = oracle.kittel_crossing_bias(
        14.29e9, MS, CONSTANTS.gamma_eff) / oersted_to_si(1.0)
    out["kittel_hz"] = {str(b): oracle.kittel_frequency(oersted_to_si(b), MS,
                                                        CONSTANTS.gamma_eff)
                        for b in BIASES_OE}
    OUT.write_text(json.dumps(out, indent=1))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
