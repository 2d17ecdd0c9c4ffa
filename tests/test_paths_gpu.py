"""GPU tests of the §8f rows: CLI simulate/sweep, energy diagnostic, bias
sweep, and a full-length acceptance-cavity run (FMR / anti-crossing path)."""

import math
from pathlib import Path

import numpy as np
import pytest

from oracle import magphon_oracle as orc
from paper_2510_22221_b200 import cli, sim
from paper_2510_22221_b200.analysis import fft_magnitude
from paper_2510_22221_b200.grid import initial_magnetization
from tests.golden.cases import CASES, build, mirror_namespace
from tests.golden_io import load

pytestmark = pytest.mark.gpu

CFG = """
[grid]
nx = 1
ny = 1
nz = 120
dx = 2 um
dy = 2 um
dz = 2 um
[background]
sigma = 1e-4 S/m
eps_r = 8.0
[material:ferrite]
box = 0 1 0 1 60 61
sigma = 1e-3 S/m
eps_r = 1.0
Ms = 9.7e5 A/m
alpha = 0.003
bias = 1855.3 Oe
[source]
f0 = 14.3 GHz
Tp = 1 ps
amplitude = 1e3 V/m
location = 0 0 10
[boundaries]
z0 = PMC
z1 = PMC
[run]
t_end = 4 ps
{extra}
[probes]
cavity = Ex 0 0 20
magnon = Mz 0 0 60
[sweep]
bias_list = 1700 Oe, 1900 Oe
"""


def test_cli_simulate_matches_oracle(tmp_path):
    cfgp = tmp_path / "c.cfg"
    cfgp.write_text(CFG.format(extra=""))
    out = tmp_path / "out"
    assert cli.main(["--out", str(out), "simulate", str(cfgp)]) == cli.EXIT_OK
    from paper_2510_22221_b200.config import load_config
    ref = orc.run(load_config(cfgp))
    for (comp, (i, j, k)), vals in ref["probes"].items():
        lines = (out / f"probe_{comp}_{i}_{j}_{k}.txt").read_text().splitlines()
        assert lines[0].startswith(f"# component={comp} i={i}")
        got = np.array([float(x) for x in lines[1:]])
        assert np.array_equal(got, np.array([float("%.12e" % v) for v in vals]))
    assert (out / "manifest.json").exists()


def test_cli_fault_injection_exit_code(tmp_path):
    cfgp = tmp_path / "f.cfg"
    cfgp.write_text(CFG.format(extra="llg_tol = 1e-16\nllg_max_iters = 1").replace(
        "amplitude = 1e3", "amplitude = 1e8"))
    assert cli.main(["--out", str(tmp_path), "simulate", str(cfgp)]) == cli.EXIT_RUNTIME


def test_sweep_matches_oracle_spectra(tmp_path):
    cfgp = tmp_path / "c.cfg"
    cfgp.write_text(CFG.format(extra=""))
    from paper_2510_22221_b200.config import load_config
    cfg = load_config(cfgp)
    smap = sim.sweep(cfg)
    for row, b in zip(smap.mags, smap.biases):
        ref = orc.run(cfg, bias=float(b))
        x = list(ref["probes"].values())[cfg.spectrum_probe]
        spec = fft_magnitude((x, ref["dt"]), window="hann")
        assert np.array_equal(row, spec.mags)
    # several concurrent runs per GPU (separate streams, host threads):
    # identical rows, in bias order
    par = sim.sweep(cfg, parallel=3)
    assert np.array_equal(par.mags, smap.mags) and np.array_equal(par.freqs, smap.freqs)


@pytest.mark.parametrize("name", ["mixed3d", "allmur3d", "pec_block"])
def test_total_energy_matches_reference_formula(name):
    case = CASES[name]
    cfg = build(case, mirror_namespace())
    res = sim.run(cfg)
    g = load(name)
    e_ref = orc.total_energy(g["fields"], cfg.materials.eps_r, cfg.materials.Hbias,
                             cfg.grid.cell_shape, cfg.grid.spacings)
    keys = [(p[0], (p[1], p[2], p[3])) for p in cfg.probes]
    dev = sim._device_run(cfg, cfg.materials, list(dict.fromkeys(keys)))
    try:
        st = res.lattice.state_arrays()
        dev.load_state({k: st[k] for k in ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")}, st["M"])
        e_dev = dev.total_energy()
    finally:
        dev.close()
    assert e_dev == pytest.approx(e_ref, rel=1e-12, abs=1e-300)


def test_acceptance_cavity_full_length_bitwise():
    """The reference acceptance testbed (test_acceptance.py:25-53): 1D cavity,
    NZ=917, DZ=4 um, one magnetic cell, 1.2 ns (~1e5 steps), strong drive so
    r* = 2 steps occur.  Probe series bit-identical => identical FFT / ESPRIT
    frequencies (north_star: within 0.1%)."""
    oe = 1000.0 / (4.0 * math.pi)
    case = dict(grid=(1, 1, 917, 4e-6, 4e-6, 4e-6),
                background=(1.2520467594271872e-4, 8.168870103908924),
                boxes=[dict(box=(0, 1, 0, 1, 458, 459), sigma=1e-3, eps_r=1.0, Ms=9.7e5,
                            alpha=0.003, bias=1855.3 * oe, bias_direction=(1, 0, 0))],
                source=dict(f0=14.3e9, Tp=50e-12, amplitude=1e6, location=(0, 0, 25),
                            polarization=(1.0, 0.0, 0.0)),
                boundaries=dict(z0="PMC", z1="PMC"), cfl=0.9, steps=99931,
                probes=[("Ex", 0, 0, 150), ("Mz", 0, 0, 458)])
    cfg = build(case, mirror_namespace())
    res = sim.run(cfg)
    ref = orc.run(cfg)
    assert np.array_equal(res.iterations, ref["iterations"])
    assert (res.iterations == 2).any()
    for key, v in ref["probes"].items():
        assert np.array_equal(res.probes[key].samples, v), key
    tail = slice(30000, None)
    a = fft_magnitude((res.probes[("Ex", (0, 0, 150))].samples[tail], cfg.dt), "hann")
    b = fft_magnitude((ref["probes"][("Ex", (0, 0, 150))][tail], ref["dt"]), "hann")
    band = (a.freqs > 10e9) & (a.freqs < 18e9)
    fa = a.freqs[band][np.argmax(a.mags[band])]
    fb = b.freqs[band][np.argmax(b.mags[band])]
    assert abs(fa - fb) <= 1e-3 * fb
