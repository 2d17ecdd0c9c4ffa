"""The CPU oracle reproduces the reference's own outputs bit for bit.

Goldens were produced by running ``magphon.sim.run`` itself
(tests/golden/make_golden.py); here the oracle is re-run on the same
configs, built through this repo's host mirror of the reference API.
"""

import numpy as np
import pytest

from oracle import magphon_oracle as orc
from tests.golden.cases import CASES, build, mirror_namespace
from tests.golden_io import load

RUNNING = [n for n in CASES if not CASES[n].get("expect_failure")]


@pytest.mark.parametrize("name", RUNNING)
def test_oracle_matches_reference_golden(name):
    case = CASES[name]
    g = load(name)
    cfg = build(case, mirror_namespace())
    assert cfg.dt == float(g["dt"]) and cfg.n_steps == int(g["steps"])
    out = orc.run(cfg, bias=case.get("bias"))
    for k, v in g["fields"].items():
        assert np.array_equal(out["fields"][k], v), k
    assert np.array_equal(out["iterations"], g["iterations"])
    for key, v in g["probes"].items():
        assert np.array_equal(out["probes"][key], v), key


def test_oracle_step_failure_matches_reference():
    g = load("fail_tol")
    cfg = build(CASES["fail_tol"], mirror_namespace())
    with pytest.raises(orc.OracleStepFailure) as ei:
        orc.run(cfg)
    assert ei.value.step == int(g["fail_step"])
    assert ei.value.iterations == int(g["fail_iterations"])
    assert ei.value.residual == float(g["fail_residual"])


def test_oracle_resume_matches_reference_snapshot():
    g = load("mixed3d_snapshot47")
    full = load("mixed3d")
    cfg = build(CASES["mixed3d"], mirror_namespace())
    snap = {"fields": g["fields"], "step": int(g["step"]),
            "probes": g["probes"], "iterations": g["iterations"]}
    out = orc.run(cfg, resume=snap)
    for k, v in full["fields"].items():
        assert np.array_equal(out["fields"][k], v), k
    assert np.array_equal(out["iterations"], full["iterations"])


def test_goldens_cover_mixed_convergence():
    # the lockstep fix-up path is only exercised when magnetic cells of one
    # step stop locally at different iterates
    assert int(load("mixed3d")["mixed_steps"]) > 0
    assert int(load("pec_block")["mixed_steps"]) > 0
    its = load("pec_block")["iterations"]
    assert set(np.unique(its)) == {1, 2}


def test_nonmonotone_golden_exercises_the_continuation():
    """nonmono3d really has steps where the reference iterates past every
    cell's own first stop (the multi-rank continuation case)."""
    g = load("nonmono3d")
    assert int(g["nonmono_steps"]) >= 2
    assert int(np.max(g["iterations"])) == 3
