"""Run-time configuration errors raised in the reference's order.

The reference raises these inside its first time step, after that step's
LLG (sim.py:151-171): MUR1 on a collapsed axis (em._capture_mur_planes),
a source index out of range (inject_soft_source), an unknown probe
component (FieldLattice.sample); with no step left to run (resume at
n_steps) it raises nothing.  Expected outcomes were read off the reference
itself (magphon.sim.run) on these exact configurations."""
from dataclasses import replace

import numpy as np
import pytest

from paper_2510_22221_b200 import llg, sim
from tests.golden.cases import CASES, build, mirror_namespace
from tests.golden_io import load

pytestmark = pytest.mark.gpu


def _cfg(name):
    return build(CASES[name], mirror_namespace())


def test_source_out_of_range_raises_index_error():
    c = _cfg("mixed3d")
    with pytest.raises(IndexError):
        sim.run(replace(c, source=replace(c.source, location=(99, 0, 0))))


def test_unknown_probe_component_raises_key_error():
    c = _cfg("mixed3d")
    with pytest.raises(KeyError):
        sim.run(replace(c, probes=c.probes + (("Qx", 1, 1, 1),)))


def test_mur1_on_collapsed_axis_raises_value_error():
    c = _cfg("small1d_strong")
    with pytest.raises(ValueError, match="MUR1 on collapsed axis"):
        sim.run(replace(c, boundaries=replace(c.boundaries, x0="MUR1")))


def test_no_step_left_no_error():
    c = _cfg("mixed3d")
    snap = sim.snapshot_state(c, None, c.n_steps)
    res = sim.run(replace(c, source=replace(c.source, location=(99, 0, 0))), resume=snap)
    assert res.steps == c.n_steps
    for k, v in snap["fields"].items():
        assert np.array_equal(res.lattice.state_arrays()[k], v), k


@pytest.mark.parametrize("broken", ["source", "mur", "probe"])
def test_first_step_llg_failure_wins(broken):
    """fail_tol resumed at its failing step (124): the reference raises the
    StepFailure of that step's LLG before the E update / source / probes."""
    f = _cfg("fail_tol")
    g = load("fail_tol")
    x = int(g["fail_step"])
    snap = sim.snapshot_state(f, None, x)
    bad = {"source": replace(f, source=replace(f.source, location=(0, 0, 999))),
           "mur": replace(f, boundaries=replace(f.boundaries, x0="MUR1")),
           "probe": replace(f, probes=f.probes + (("Qx", 0, 0, 1),))}[broken]
    with pytest.raises(llg.StepFailure) as ei:
        sim.run(bad, resume=snap)
    assert ei.value.step == x
    assert ei.value.iterations == int(g["fail_iterations"])
    assert ei.value.residual == float(g["fail_residual"])
