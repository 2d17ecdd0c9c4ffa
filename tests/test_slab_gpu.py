"""Multi-rank x-slab decomposition, emulated on one GPU (mpb_group_run):
the same kernels and boundary-plane movement as the NCCL path must give
results bit-identical to the reference goldens (SURVEY 8e correctness gate:
P-rank == 1-rank, bitwise)."""

import numpy as np
import pytest

from paper_2510_22221_b200 import parallel
from tests.golden.cases import CASES, build, mirror_namespace
from tests.golden_io import load

pytestmark = pytest.mark.gpu

SPLITS = [("mixed3d", 2), ("mixed3d", 3), ("allmur3d", 2), ("allmur3d", 5),
          ("pec_block", 4), ("zwall_magnet", 2), ("zwall_magnet", 3), ("thin", 3),
          ("plane2d", 2), ("xline1d", 4), ("bias3d", 2), ("plane_xz", 3),
          ("cpw_small", 3), ("two_magnets", 2), ("two_magnets", 4),
          # global residual non-monotone past the last local stop: the
          # suspended step is continued in lockstep on the host
          ("nonmono3d", 2), ("nonmono3d", 3)]


@pytest.mark.parametrize("name,nranks", SPLITS)
def test_slab_group_matches_reference_golden(name, nranks):
    case = CASES[name]
    g = load(name)
    cfg = build(case, mirror_namespace())
    fields, M, probes, its = parallel.run_group(cfg, nranks, bias=case.get("bias"))
    assert fields is not None, f"step failure: {its}"
    for k, v in g["fields"].items():
        got = M if k == "M" else fields[k]
        assert np.array_equal(got, v), (k, np.max(np.abs(got - v)))
    assert np.array_equal(its, g["iterations"])
    for key, v in g["probes"].items():
        assert np.array_equal(probes[key], v), key


# Short x-chunks (2 planes) give every slab >= 3 chunks, so the overlapped
# path really splits each sweep into interior chunks (running while the
# previous step's boundary copies are in flight on the comm stream) and edge
# chunks (after them); MPB_OVERLAP=0 is the serialised order.
@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("name,nranks", [("mixed3d", 2), ("pec_block", 2), ("bias3d", 2),
                                         ("allmur3d", 2), ("nonmono3d", 2)])
def test_slab_overlapped_exchange_matches_golden(name, nranks, overlap, monkeypatch):
    monkeypatch.setenv("MPB_SWEEP_MINCHUNK", "2")
    monkeypatch.setenv("MPB_OVERLAP", overlap)
    test_slab_group_matches_reference_golden(name, nranks)


# Benchmark-size geometries in slabs: C2 (CPW + film, the C4 geometry family)
# and C3 (7% magnetic film) from a mid-run state, 3 and 4 slabs with many
# x-chunks each (interior/edge split of the overlapped exchange) against the
# single-GPU run of the same state (itself bit-identical to the oracle,
# tests/test_configs_gpu.py).
@pytest.mark.parametrize("name,nranks,steps", [("c2", 3, 6), ("c3", 4, 4)])
def test_slab_group_benchmark_geometry(name, nranks, steps):
    from dataclasses import replace
    from pathlib import Path

    from paper_2510_22221_b200 import sim
    from paper_2510_22221_b200.config import load_config
    from tests.test_configs_gpu import mid_run_state

    cfg = load_config(Path(__file__).resolve().parents[1] / "configs" / f"{name}.cfg")
    start = 200
    cfg = replace(cfg, t_end=(start + steps - 0.5) * cfg.dt)
    state = mid_run_state(cfg, 11)
    keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in cfg.probes))
    snap = {"fields": {k: v.copy() for k, v in state.items()}, "step": start,
            "probes": {k: np.zeros(start) for k in keys},
            "iterations": np.ones(start, dtype=int)}
    one = sim.run(cfg, resume=snap)
    fields, M, probes, its = parallel.run_group(cfg, nranks, state=state, start=start)
    assert fields is not None, its
    st = one.lattice.state_arrays()
    for k in ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz"):
        assert np.array_equal(fields[k], st[k]), k
    assert np.array_equal(M, st["M"])
    assert np.array_equal(its, one.iterations[start:])
    for key in keys:
        assert np.array_equal(probes[key], one.probes[key].samples[start:]), key



@pytest.mark.parametrize("nranks", [2, 3])
def test_slab_group_step_failure(nranks):
    """The global stop rule fails across slabs exactly where the reference
    raises StepFailure (same step, residual, iterate count)."""
    g = load("fail3d")
    cfg = build(CASES["fail3d"], mirror_namespace())
    fields, M, probes, fail = parallel.run_group(cfg, nranks)
    assert fields is None
    step, residual, iterations, kind = fail
    assert step == int(g["fail_step"])
    assert residual == float(g["fail_residual"])
    assert iterations == int(g["fail_iterations"])


@pytest.mark.parametrize("nranks", [2, 3])
def test_slab_group_continues_nonmonotone_steps(nranks):
    """nonmono3d's steps 6 and 14 have a global residual back above tol after
    every cell's own stop: the reference iterates on (llg.py:131-148), and
    the slab path must suspend and continue exactly those steps."""
    g = load("nonmono3d")
    cfg = build(CASES["nonmono3d"], mirror_namespace())
    stats = {}
    fields, M, probes, its = parallel.run_group(cfg, nranks, stats=stats)
    assert fields is not None, its
    assert stats["continued_steps"] == int(g["nonmono_steps"]) == 2
    assert np.array_equal(its, g["iterations"])
    assert np.array_equal(M, g["fields"]["M"])
