"""CUDA path vs reference goldens and the CPU oracle -- bit for bit.

All goldens come from the reference itself (tests/golden/make_golden.py).
Tolerance: none -- fp64 results must be identical (np.array_equal), which
is stricter than north_star's rel-L2 <= 1e-10.
"""

import numpy as np
import pytest

from oracle import magphon_oracle as orc
from paper_2510_22221_b200 import llg, sim
from tests.golden.cases import CASES, build, mirror_namespace
from tests.golden_io import load

pytestmark = pytest.mark.gpu

VARIANTS = [0, 1]
RUNNING = [n for n in CASES if not CASES[n].get("expect_failure")]


def _assert_same(res, g):
    for k, v in g["fields"].items():
        got = res.lattice.state_arrays()[k]
        assert np.array_equal(got, v), (k, np.max(np.abs(got - v)))
    assert np.array_equal(res.iterations, g["iterations"])
    for key, v in g["probes"].items():
        assert np.array_equal(res.probes[key].samples, v), key


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("name", RUNNING)
def test_gpu_matches_reference_golden(name, variant):
    case = CASES[name]
    cfg = build(case, mirror_namespace())
    res = sim.run(cfg, bias=case.get("bias"), kernel_variant=variant)
    assert res.steps == int(load(name)["steps"])
    _assert_same(res, load(name))


@pytest.mark.parametrize("name", ["fail_tol", "fail3d"])
@pytest.mark.parametrize("variant", VARIANTS)
def test_gpu_step_failure(variant, name):
    g = load(name)
    cfg = build(CASES[name], mirror_namespace())
    with pytest.raises(llg.StepFailure) as ei:
        sim.run(cfg, kernel_variant=variant)
    assert ei.value.step == int(g["fail_step"])
    assert ei.value.iterations == int(g["fail_iterations"])
    assert ei.value.residual == float(g["fail_residual"])
    assert str(ei.value) == str(g["fail_message"])


@pytest.mark.parametrize("variant", VARIANTS)
def test_gpu_resume_from_reference_snapshot(variant):
    g = load("mixed3d_snapshot47")
    cfg = build(CASES["mixed3d"], mirror_namespace())
    snap = {"fields": g["fields"], "step": int(g["step"]), "probes": g["probes"],
            "iterations": g["iterations"]}
    _assert_same(sim.run(cfg, resume=snap, kernel_variant=variant), load("mixed3d"))


def test_gpu_snapshot_roundtrip(tmp_path):
    cfg = build(CASES["pec_block"], mirror_namespace())
    snap = sim.snapshot_state(cfg, None, 61)
    sim.save_snapshot(tmp_path / "s.npz", snap)
    back = sim.load_snapshot(tmp_path / "s.npz")
    _assert_same(sim.run(cfg, resume=back), load("pec_block"))


def test_gpu_deterministic_repeat():
    cfg = build(CASES["allmur3d"], mirror_namespace())
    a, b = sim.run(cfg), sim.run(cfg)
    for k, v in a.lattice.state_arrays().items():
        assert np.array_equal(v, b.lattice.state_arrays()[k])


C1_VARIANTS = {
    "weak": 1e3, "medium": 1e6, "strong": 1e8,
}


@pytest.mark.parametrize("amp", sorted(C1_VARIANTS))
def test_gpu_c1_64cubed_against_oracle(amp):
    """C1: 64^3 PEC box, YIG block 28:36, 300 steps, vs the
    oracle run live on this host."""
    case = dict(
        grid=(64, 64, 64, 10e-6, 10e-6, 10e-6), background=(0.0, 1.0),
        boxes=[dict(box=(28, 36, 28, 36, 28, 36), eps_r=15.0,
                    Ms=1750.0 * 1000.0 / (4 * np.pi), alpha=1e-3,
                    bias=1000.0 * 1000.0 / (4 * np.pi), bias_direction=(0, 0, 1))],
        source=dict(f0=50e9, Tp=1e-12, amplitude=C1_VARIANTS[amp],
                    location=(16, 32, 32), polarization=(0.0, 1.0, 0.0)),
        boundaries=dict(x0="PEC", x1="PEC", y0="PEC", y1="PEC", z0="PEC", z1="PEC"),
        cfl=0.9, steps=300,
        probes=[("Ey", 17, 32, 32), ("Hx", 32, 32, 32), ("Mx", 32, 32, 32),
                ("My", 32, 32, 32), ("Mz", 32, 32, 32)])
    cfg = build(case, mirror_namespace())
    res = sim.run(cfg)
    ref = orc.run(cfg)
    for k, v in ref["fields"].items():
        assert np.array_equal(res.lattice.state_arrays()[k], v), k
    assert np.array_equal(res.iterations, ref["iterations"])
    for key, v in ref["probes"].items():
        assert np.array_equal(res.probes[key].samples, v), key


# z walls as separate launches instead of inside the sweep (MPB_ZWALL=kernel):
# the other documented order of the same wall arithmetic, same bits
@pytest.mark.parametrize("name", ["mixed3d", "allmur3d", "zwall_magnet", "pec_block"])
def test_gpu_zwall_kernel_order_matches_golden(name, monkeypatch):
    monkeypatch.setenv("MPB_ZWALL", "kernel")
    case = CASES[name]
    res = sim.run(build(case, mirror_namespace()), bias=case.get("bias"))
    _assert_same(res, load(name))


# Plain stream-ordered launches instead of programmatic dependent launch
# (MPB_PDL=0): the same kernels with full serialisation, same bits.
@pytest.mark.parametrize("name", ["mixed3d", "allmur3d", "two_magnets"])
def test_gpu_without_pdl_matches_golden(name, monkeypatch):
    monkeypatch.setenv("MPB_PDL", "0")
    case = CASES[name]
    res = sim.run(build(case, mirror_namespace()), bias=case.get("bias"))
    _assert_same(res, load(name))


# Lines along z run in the shared-memory line kernel by default (k_line);
# the general kernels must still give the same bits for them (MPB_LINE=0),
# including the StepFailure case.
@pytest.mark.parametrize("name", ["cavity1d", "small1d_strong"])
def test_gpu_line_general_path_matches_golden(name, monkeypatch):
    monkeypatch.setenv("MPB_LINE", "0")
    case = CASES[name]
    _assert_same(sim.run(build(case, mirror_namespace()), bias=case.get("bias")), load(name))


def test_gpu_line_general_path_step_failure(monkeypatch):
    monkeypatch.setenv("MPB_LINE", "0")
    g = load("fail_tol")
    cfg = build(CASES["fail_tol"], mirror_namespace())
    with pytest.raises(llg.StepFailure) as ei:
        sim.run(cfg)
    assert ei.value.step == int(g["fail_step"])
    assert str(ei.value) == str(g["fail_message"])


# Single-rank runs compute the magnetic cells' LLG before the sweep (the
# LLG-first order, k_llg_pre); MPB_LLG_PRE=0 keeps the order multi-rank runs
# use (sweep, k_llg_local, k_llg_fixup, deferred E).  Both give the same bits.
@pytest.mark.parametrize("name", RUNNING)
def test_gpu_llg_after_sweep_order_matches_golden(name, monkeypatch):
    monkeypatch.setenv("MPB_LLG_PRE", "0")
    case = CASES[name]
    _assert_same(sim.run(build(case, mirror_namespace()), bias=case.get("bias")), load(name))


@pytest.mark.parametrize("name", ["fail_tol", "fail3d"])
def test_gpu_llg_after_sweep_order_step_failure(name, monkeypatch):
    monkeypatch.setenv("MPB_LLG_PRE", "0")
    g = load(name)
    with pytest.raises(llg.StepFailure) as ei:
        sim.run(build(CASES[name], mirror_namespace()))
    assert ei.value.step == int(g["fail_step"])
    assert ei.value.iterations == int(g["fail_iterations"])
    assert ei.value.residual == float(g["fail_residual"])


# LLG-first order as two launches (k_llg_pre with programmatic launch, then
# the cooperative k_llg_fixup) instead of the default single cooperative one.
@pytest.mark.parametrize("name", ["mixed3d", "two_magnets", "nonmono3d", "bias3d", "cpw_small"])
def test_gpu_llg_pre_two_launch_form_matches_golden(name, monkeypatch):
    monkeypatch.setenv("MPB_LLG_COOP", "0")
    case = CASES[name]
    _assert_same(sim.run(build(case, mirror_namespace()), bias=case.get("bias")), load(name))


@pytest.mark.parametrize("name", ["fail_tol", "fail3d"])
def test_gpu_llg_pre_two_launch_form_step_failure(name, monkeypatch):
    monkeypatch.setenv("MPB_LLG_COOP", "0")
    g = load(name)
    with pytest.raises(llg.StepFailure) as ei:
        sim.run(build(CASES[name], mirror_namespace()))
    assert ei.value.step == int(g["fail_step"])
    assert ei.value.iterations == int(g["fail_iterations"])
    assert ei.value.residual == float(g["fail_residual"])
