"""The benchmark geometries on the CUDA path vs the CPU
oracle, bit for bit, from a mid-run state.

A fresh run is exact zeros almost everywhere for thousands of steps, so each
case resumes from a synthetic mid-run state: random E/H on every physical
entry (allocation padding stays zero, as in any real run) and M tilted away
from the bias in the magnetic cells, which makes the LLG fixed point take
several iterates.  Then K steps on the GPU and in the oracle, compared with
np.array_equal (fields, M, probes, r* per step).
"""
from dataclasses import replace
from pathlib import Path

import numpy as np
import pytest

from oracle import magphon_oracle as orc
from paper_2510_22221_b200 import sim
from paper_2510_22221_b200.config import load_config

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

# physical (non-padding) extent of each component, in cells (+1 = node axis)
_EXTENT = {"Ex": (0, 1, 1), "Ey": (1, 0, 1), "Ez": (1, 1, 0),
           "Hx": (1, 0, 0), "Hy": (0, 1, 0), "Hz": (0, 0, 1)}


def mid_run_state(cfg, seed):
    g = cfg.grid
    n = (g.nx, g.ny, g.nz)
    rng = np.random.default_rng(seed)
    fields = {}
    for name, ext in _EXTENT.items():
        a = np.zeros(tuple(x + 1 for x in n))
        sl = tuple(slice(0, n[ax] + ext[ax]) for ax in range(3))
        scale = 1e3 if name[0] == "E" else 2.65
        a[sl] = rng.standard_normal(a[sl].shape) * scale
        fields[name] = a
    Ms = np.asarray(cfg.materials.Ms)
    Hb = np.asarray(cfg.materials.Hbias)
    M = np.zeros((3,) + n)
    mag = Ms > 0
    hn = np.sqrt(Hb[0] ** 2 + Hb[1] ** 2 + Hb[2] ** 2)
    for c in range(3):
        u = np.where(mag, Hb[c] / np.where(hn > 0, hn, 1.0), 0.0)
        M[c] = Ms * (u + 0.05 * rng.standard_normal(n) * mag)
    nrm = np.sqrt(M[0] ** 2 + M[1] ** 2 + M[2] ** 2)
    M = np.where(mag, M * Ms / np.where(nrm > 0, nrm, 1.0), 0.0)
    fields["M"] = M
    return fields


_ORACLE = {}


def _case(name, steps):
    cfg = load_config(ROOT / "configs" / f"{name}.cfg")
    start = 200
    dt = orc.cfl_dt((cfg.grid.nx, cfg.grid.ny, cfg.grid.nz),
                    (cfg.grid.dx, cfg.grid.dy, cfg.grid.dz), cfg.cfl_factor)
    cfg = replace(cfg, t_end=(start + steps - 0.5) * dt)
    keys = [(p[0], (p[1], p[2], p[3])) for p in cfg.probes]
    any_mag = bool(np.any(np.asarray(cfg.materials.Ms) > 0))
    snap = {"fields": mid_run_state(cfg, 7), "step": start,
            "probes": {k: np.zeros(start) for k in keys},
            "iterations": np.ones(start, dtype=int) if any_mag else np.zeros(0, dtype=int)}
    if (name, steps) not in _ORACLE:
        _ORACLE[(name, steps)] = orc.run(
            cfg, resume={**snap, "fields": {k: v.copy() for k, v in snap["fields"].items()}})
    return cfg, snap, _ORACLE[(name, steps)], any_mag, start


def _check(name, steps):
    cfg, snap, ref, any_mag, start = _case(name, steps)
    res = sim.run(cfg, resume=snap)
    assert res.steps == ref["steps"] == start + steps
    for k, v in ref["fields"].items():
        got = res.lattice.state_arrays()[k]
        assert np.array_equal(got, v), (k, float(np.max(np.abs(got - v))))
    assert np.array_equal(res.iterations, ref["iterations"])
    if any_mag:
        assert int(np.max(ref["iterations"][start:])) >= 2   # non-trivial fixed point
    for key, v in ref["probes"].items():
        assert np.array_equal(res.probes[key].samples, v), key


@pytest.mark.parametrize("name,steps", [("c1", 8), ("c2", 6), ("c3", 4)])
def test_config_geometry_matches_oracle(name, steps):
    _check(name, steps)


# every sweep instantiation (entries per thread V x CTA size NT) and odd tile
# sizes must give the same bits: the tile shape is chosen per grid at setup
@pytest.mark.parametrize("env", [
    {"MPB_SWEEP_NT": "512"},                       # V=2, one 512-thread CTA per SM (C5 form)
    {"MPB_SWEEP_V": "1"},                          # one entry per thread
    {"MPB_SWEEP_T": "334", "MPB_SWEEP_MINCHUNK": "3"},   # ragged tiles and chunks
    {"MPB_SWEEP_CHUNKS": "128"},                   # two-plane chunks (the C1 choice)
])
def test_sweep_tile_forms_match_oracle(env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _check("c2", 6)


# the LLG launch forms: cooperative LLG overlapped with the sweep (default:
# only the sweep CTAs staging magnetic H wait for the LLG's step stamp), the
# cooperative LLG followed by a plain sweep, and two launches (local LLG +
# fixup) -- same bits
@pytest.mark.parametrize("env", [{}, {"MPB_LLG_OVERLAP": "1"}, {"MPB_LLG_OVERLAP": "0"},
                                 {"MPB_LLG_COOP": "0"}])
@pytest.mark.parametrize("name,steps", [("c1", 8), ("c3", 4)])
def test_llg_launch_forms_match_oracle(name, steps, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _check(name, steps)


def test_nonzero_m_outside_magnets_is_preserved():
    """A resumed state may carry M in non-magnetic cells (the reference never
    touches it there); the library keeps such planes on the host and must hand
    them back unchanged, bit for bit with the oracle."""
    cfg = load_config(ROOT / "configs" / "c2.cfg")
    start, steps = 50, 3
    cfg = replace(cfg, t_end=(start + steps - 0.5) * cfg.dt)
    state = mid_run_state(cfg, 3)
    rng = np.random.default_rng(5)
    mag = np.asarray(cfg.materials.Ms) > 0
    state["M"] = np.where(mag, state["M"], rng.standard_normal(state["M"].shape))
    keys = [(p[0], (p[1], p[2], p[3])) for p in cfg.probes]
    snap = {"fields": state, "step": start, "probes": {k: np.zeros(start) for k in keys},
            "iterations": np.ones(start, dtype=int)}
    ref = orc.run(cfg, resume={**snap, "fields": {k: v.copy() for k, v in state.items()}})
    res = sim.run(cfg, resume=snap)
    for k, v in ref["fields"].items():
        assert np.array_equal(res.lattice.state_arrays()[k], v), k
    for key, v in ref["probes"].items():
        assert np.array_equal(res.probes[key].samples, v), key


def test_guard_free_h_phase_is_bitwise_through_a_run_from_rest(monkeypatch):
    """The sweep's H phase skips the exact-division guard only while a
    per-step flag proves every E value in range (kSafeBias); a run from rest
    goes through zeros and a shell of tiny values ahead of its wavefront, so
    the flag switches both ways.  Same bits as with the guard always on."""
    cfg = load_config(ROOT / "configs" / "c3.cfg")
    cfg = replace(cfg, t_end=(400 - 0.5) * cfg.dt)
    a = sim.run(cfg)
    monkeypatch.setenv("MPB_EGUARD", "0")
    b = sim.run(cfg)
    for k, v in b.lattice.state_arrays().items():
        assert np.array_equal(a.lattice.state_arrays()[k], v), k
    for key, v in b.probes.items():
        assert np.array_equal(a.probes[key].samples, v.samples), key


def test_concurrent_overlapped_runs_match_oracle():
    """Four C1 runs at once on one GPU (host threads, one handle + stream
    each; the C ABI releases the GIL), each with the sweep overlapping its
    cooperative LLG: CTAs spinning on one handle's step stamp must never
    hold up another handle's LLG, and every run gives the oracle's bits."""
    from concurrent.futures import ThreadPoolExecutor
    cfg, snap, ref, any_mag, start = _case("c1", 8)
    assert any_mag

    def one(_):
        return sim.run(cfg, resume={**snap, "fields": {k: v.copy()
                                                        for k, v in snap["fields"].items()}})

    with ThreadPoolExecutor(4) as ex:
        results = list(ex.map(one, range(4)))
    for res in results:
        for k, v in ref["fields"].items():
            assert np.array_equal(res.lattice.state_arrays()[k], v), k
        assert np.array_equal(res.iterations, ref["iterations"])
        for key, v in ref["probes"].items():
            assert np.array_equal(res.probes[key].samples, v), key
