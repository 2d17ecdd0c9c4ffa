"""The reference's own physics and run-loop tests, re-run on the CUDA path.

The reference pins its solver with behavioural tests (pkg/tests/test_em.py,
test_simulation.py): causality at the magic time step, bounded energy in a
closed box, PEC zeroing, the PMC cavity frequency, MUR1 absorption, ohmic
decay, probes/iterations bookkeeping, bias override, restart.  The goldens
already show the CUDA path is bit-identical to the reference on small cases;
these tests check the same physical statements the reference checks, at the
reference's sizes and step counts, on the device (the per-step source and
energy read-outs go through the engine, i.e. the C ABI).
"""
import math

import numpy as np
import pytest

from paper_2510_22221_b200 import em, sim
from paper_2510_22221_b200.constants import CONSTANTS, oersted_to_si
from paper_2510_22221_b200.grid import GridSpec, initial_magnetization
from paper_2510_22221_b200.materials import MaterialCell, MaterialMap

pytestmark = pytest.mark.gpu

C0 = 299792458.0


def line_config(nz, dz, cfl, faces=None, src=None, probes=(), background=None, magnet=None,
                steps=1):
    """1D line along z (the reference tests' geometry)."""
    grid = GridSpec(1, 1, nz, dz, dz, dz)
    mm = MaterialMap(grid.cell_shape, background or MaterialCell())
    if magnet is not None:
        mm.fill_box(*magnet)
    mm.freeze()
    dt = em.cfl_timestep(grid, cfl)
    return sim.SimConfig(grid=grid, materials=mm,
                         source=src or em.SourceSpec(amplitude=0.0),
                         boundaries=em.BoundarySpec(**(faces or {})),
                         cfl_factor=cfl, t_end=(steps - 0.5) * dt, probes=tuple(probes))


class Stepper:
    """Device state of one config, advanced in chunks with explicit source
    values (lets a test switch the source off like the reference tests do)."""

    def __init__(self, cfg):
        self.cfg = cfg
        self.keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in cfg.probes))
        self.dev = sim._device_run(cfg, cfg.materials, self.keys)
        z = np.zeros(cfg.grid.field_shape)
        self.dev.load_state({n: z for n in ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")},
                            initial_magnetization(cfg.materials))
        self.n = 0

    def advance(self, steps, source_on=True):
        vals = sim.source_values(self.cfg.source, self.cfg.dt, self.n, self.n + steps)
        if not source_on:
            vals[:] = 0.0
        probes, iters, fail = self.dev.run(self.n, vals)
        assert fail is None
        self.n += steps
        return probes

    def energy(self):
        return self.dev.total_energy()

    def state(self):
        return self.dev.save_state()

    def close(self):
        self.dev.close()


def test_magic_timestep_causality_1d():
    """At the CFL limit in 1D the front moves exactly one cell per step."""
    cfg = line_config(400, 1e-6, 1.0,
                      src=em.SourceSpec(f0=50e9, Tp=20e-12, amplitude=1.0,
                                        location=(0, 0, 100), polarization=(1, 0, 0)),
                      steps=150)
    ex = sim.run(cfg).lattice.state_arrays()["Ex"][0, 0]
    assert np.all(ex[100 + 150 + 1:] == 0.0)
    assert np.abs(ex[100:250]).max() > 1e-3


def test_closed_box_energy_bounded_10k_steps():
    cfg = line_config(400, 1e-6, 0.99,
                      src=em.SourceSpec(f0=100e9, Tp=1e-12, amplitude=1.0,
                                        location=(0, 0, 100), polarization=(1, 0, 0)))
    st = Stepper(cfg)
    try:
        st.advance(2500)
        energies = []
        for _ in range(7500 // 25):
            st.advance(25, source_on=False)
            energies.append(st.energy())
    finally:
        st.close()
    e = np.asarray(energies)
    drift = abs(e[-8:].mean() - e[:8].mean()) / e[:8].mean()
    assert drift < 1e-3
    assert e.max() / e.min() < 1.05


def test_pec_wall_zeroes_tangential_e_every_step():
    cfg = line_config(50, 1e-6, 0.9,
                      src=em.SourceSpec(f0=100e9, Tp=2e-12, amplitude=1.0,
                                        location=(0, 0, 25), polarization=(1, 0, 0)),
                      probes=[("Ex", 0, 0, 0), ("Ex", 0, 0, 50), ("Ex", 0, 0, 24)],
                      steps=400)
    res = sim.run(cfg)
    assert np.all(res.probes[("Ex", (0, 0, 0))].samples == 0.0)
    assert np.all(res.probes[("Ex", (0, 0, 50))].samples == 0.0)
    assert np.abs(res.probes[("Ex", (0, 0, 24))].samples).max() > 0.0


def test_pmc_cavity_fundamental_frequency():
    nz, dz = 200, 1e-6
    f_exp = C0 / (2 * nz * dz)                  # PMC-PMC cavity: c / 2L
    cfg = line_config(nz, dz, 0.9, faces=dict(z0="PMC", z1="PMC"),
                      src=em.SourceSpec(f0=f_exp, Tp=1.0 / f_exp, amplitude=1.0,
                                        location=(0, 0, 30), polarization=(1, 0, 0)),
                      probes=[("Ex", 0, 0, 77)])
    st = Stepper(cfg)
    try:
        rec = np.concatenate([st.advance(4000)[:, 0], st.advance(8000, source_on=False)[:, 0]])
    finally:
        st.close()
    x = rec[5000:]
    freqs = np.fft.rfftfreq(len(x), cfg.dt)
    f_peak = freqs[np.argmax(np.abs(np.fft.rfft(x * np.hanning(len(x)))))]
    assert f_peak == pytest.approx(f_exp, rel=0.02)


@pytest.mark.parametrize("cfl,bound", [(1.0, 1e-6), (0.9, 0.08)])
def test_mur1_absorbs_outgoing_pulse(cfl, bound):
    """First-order Mur walls: exact at the 1D magic step, ~5% reflection at
    0.9 CFL.  The residue is measured on node averages (the soft source also
    leaves a stationary Nyquist checkerboard no wall can drain)."""
    nz = 600
    cfg = line_config(nz, 1e-6, cfl, faces=dict(z0="MUR1", z1="MUR1"),
                      src=em.SourceSpec(f0=30e9, Tp=3e-12, amplitude=1.0,
                                        location=(0, 0, 300), polarization=(1, 0, 0)),
                      probes=[("Ex", 0, 0, k) for k in range(nz + 1)], steps=9000)
    res = sim.run(cfg)
    peak = max(np.abs(res.probes[("Ex", (0, 0, k))].samples).max() for k in range(nz + 1))
    st = res.lattice.state_arrays()
    ex, hy = st["Ex"][0, 0], st["Hy"][0, 0, :-1]
    eta0 = math.sqrt(CONSTANTS.mu0 / CONSTANTS.eps0)
    residual = max(np.abs(0.5 * (ex[1:] + ex[:-1])).max(),
                   eta0 * np.abs(0.5 * (hy[1:] + hy[:-1])).max())
    assert residual < bound * peak


def test_conductive_loss_decays_energy():
    cfg = line_config(100, 1e-6, 0.9, faces=dict(z0="PMC", z1="PMC"),
                      background=MaterialCell(sigma=5.0),
                      src=em.SourceSpec(f0=100e9, Tp=2e-12, amplitude=1.0,
                                        location=(0, 0, 50), polarization=(1, 0, 0)))
    st = Stepper(cfg)
    try:
        st.advance(100)
        st.advance(200, source_on=False)
        e_mid = st.energy()
        st.advance(3000, source_on=False)
        e_end = st.energy()
    finally:
        st.close()
    assert e_end < 0.5 * e_mid


def _cavity(nz=120, steps=None, t_end=4e-12, magnet=True):
    """The reference run-loop tests' cavity: lossy dielectric line, PMC ends,
    one YIG cell in the middle biased along x."""
    grid = GridSpec(1, 1, nz, 2e-6, 2e-6, 2e-6)
    mm = MaterialMap(grid.cell_shape, MaterialCell(sigma=1e-4, eps_r=8.0))
    if magnet:
        mm.fill_box(MaterialCell(sigma=1e-3, eps_r=1.0, Ms=9.7e5, alpha=0.003,
                                 Hbias=(oersted_to_si(1855.3), 0.0, 0.0)),
                    0, 1, 0, 1, nz // 2, nz // 2 + 1)
    mm.freeze()
    return sim.SimConfig(
        grid=grid, materials=mm,
        source=em.SourceSpec(f0=14.3e9, Tp=1e-12, amplitude=1e3, location=(0, 0, 10),
                             polarization=(1, 0, 0)),
        boundaries=em.BoundarySpec(z0="PMC", z1="PMC"), cfl_factor=0.9, t_end=t_end,
        probes=(("Ex", 0, 0, 20), ("Mz", 0, 0, nz // 2)), bias_direction=(1.0, 0.0, 0.0))


def test_run_records_probes_and_iterations():
    cfg = _cavity()
    res = sim.run(cfg)
    assert res.steps == cfg.n_steps
    ex, mz = res.probes[("Ex", (0, 0, 20))], res.probes[("Mz", (0, 0, 60))]
    assert len(ex) == len(mz) == res.steps
    assert ex.dt_sample == cfg.dt
    assert np.abs(ex.samples).max() > 0.0
    assert res.iterations.shape == (res.steps,) and res.iterations.max() >= 1
    assert sim.run(_cavity(magnet=False)).iterations.size == 0


def test_bias_override_changes_magnon_dynamics():
    cfg = _cavity(t_end=8e-12)
    lo = sim.run(cfg, bias=oersted_to_si(1000.0))
    hi = sim.run(cfg, bias=oersted_to_si(2400.0))
    assert lo.bias != hi.bias
    a, b = lo.probes[("Mz", (0, 0, 60))].samples, hi.probes[("Mz", (0, 0, 60))].samples
    assert np.abs(a - b).max() > 0.0


def test_snapshot_resume_is_bit_identical(tmp_path):
    cfg = _cavity(t_end=6e-12)
    bias = oersted_to_si(1855.3)
    full = sim.run(cfg, bias=bias)
    snap = sim.snapshot_state(cfg, bias, until_step=cfg.n_steps // 2)
    sim.save_snapshot(tmp_path / "snap.npz", snap)
    resumed = sim.run(cfg, bias=bias, resume=sim.load_snapshot(tmp_path / "snap.npz"))
    for key, series in full.probes.items():
        assert np.array_equal(resumed.probes[key].samples, series.samples)
    assert np.array_equal(resumed.iterations, full.iterations)
    for name, arr in full.lattice.state_arrays().items():
        assert np.array_equal(resumed.lattice.state_arrays()[name], arr)


def test_closed_box_energy_bounded_3d_long_run():
    """3D counterpart of the closed-box check (reference test_em.py:99-113):
    a vacuum PEC box at 0.99 CFL, pulse injected then switched off, 20,000
    steps; the on-device total_energy must neither drift (< 1e-3) nor
    oscillate beyond 5% -- long-run stability of the fused 3D sweep."""
    grid = GridSpec(24, 20, 28, 1e-6, 1.2e-6, 0.9e-6)
    mm = MaterialMap(grid.cell_shape, MaterialCell()).freeze()
    dt = em.cfl_timestep(grid, 0.99)
    cfg = sim.SimConfig(grid=grid, materials=mm,
                        source=em.SourceSpec(f0=150e9, Tp=0.5e-12, amplitude=1.0,
                                             location=(7, 9, 11), polarization=(0, 1, 0)),
                        boundaries=em.BoundarySpec(), cfl_factor=0.99,
                        t_end=0.5 * dt, probes=())
    st = Stepper(cfg)
    try:
        st.advance(1500)
        energies = []
        for _ in range(185):
            st.advance(100, source_on=False)
            energies.append(st.energy())
    finally:
        st.close()
    e = np.asarray(energies)
    assert e.min() > 0
    drift = abs(e[-10:].mean() - e[:10].mean()) / e[:10].mean()
    assert drift < 1e-3
    assert e.max() / e.min() < 1.05
