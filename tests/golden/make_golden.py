"""Generate the golden parity fixtures from the REAL reference.

Run in the build container (it needs /root/reference; the GPU box does not):

    python tests/golden/make_golden.py

For every case in ``cases.py`` it runs ``magphon.sim.run`` (the reference
itself) and the CPU oracle (``oracle/magphon_oracle.py``) on the same config,
asserts they agree bit for bit, and writes ``tests/golden/<case>.npz`` with
the reference's final E/H/M, probe series, LLG iteration counts (or the
StepFailure record).  It also stores a snapshot/resume golden and checks the
config loader of this repo against the reference loader.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from oracle import magphon_oracle as orc  # noqa: E402
from tests.golden.cases import CASES, build, mirror_namespace, reference_namespace  # noqa: E402

OUT = Path(__file__).resolve().parent


def _probe_key(k):
    comp, (i, j, kk) = k
    return f"probe__{comp}__{i}__{j}__{kk}"


def main() -> None:
    from magphon import llg as rllg
    from magphon import sim as rsim

    rns, mns = reference_namespace(), mirror_namespace()
    only = sys.argv[1:]           # optional case names: regenerate just those
    for name, case in CASES.items():
        if only and name not in only:
            continue
        rcfg = build(case, rns)
        mcfg = build(case, mns)
        bias = case.get("bias")
        payload = {"dt": np.float64(rcfg.dt), "steps": np.int64(rcfg.n_steps)}
        try:
            ref = rsim.run(rcfg, bias=bias)
            failed = None
        except rllg.StepFailure as exc:
            ref, failed = None, exc
        if failed is not None:
            try:
                orc.run(mcfg, bias=bias)
                raise AssertionError(f"{name}: oracle did not fail")
            except orc.OracleStepFailure as exc:
                assert (exc.step, exc.iterations) == (failed.step, failed.iterations)
                assert np.array_equal(exc.residual, failed.residual)
            payload.update(fail_step=np.int64(failed.step),
                           fail_residual=np.float64(failed.residual),
                           fail_iterations=np.int64(failed.iterations),
                           fail_message=np.str_(str(failed)))
            print(f"{name}: StepFailure at step {failed.step} ({failed})")
        else:
            mine = orc.run(mcfg, bias=bias, record_first=True)
            for k, v in ref.lattice.state_arrays().items():
                assert np.array_equal(v, mine["fields"][k]), (name, k)
                payload["field__" + k] = v
            assert np.array_equal(ref.iterations, mine["iterations"]), name
            payload["iterations"] = ref.iterations
            for key, ser in ref.probes.items():
                assert np.array_equal(ser.samples, mine["probes"][key]), (name, key)
                payload[_probe_key(key)] = ser.samples
            mixed = sum(int(len(set(f.tolist())) > 1) for f in mine["first_converged"])
            payload["mixed_steps"] = np.int64(mixed)
            # steps whose r* exceeds every cell's own first stop: the global
            # residual went back above tol after the last local stop
            nonmono = sum(int(f.size and int(f.max()) < int(r))
                          for f, r in zip(mine["first_converged"], ref.iterations))
            payload["nonmono_steps"] = np.int64(nonmono)
            its = ref.iterations
            print(f"{name}: {ref.steps} steps, r* histogram "
                  f"{dict(zip(*np.unique(its, return_counts=True))) if its.size else {}}, "
                  f"steps with per-cell stop disagreement: {mixed}, non-monotone: {nonmono}")
        np.savez_compressed(OUT / f"{name}.npz", **payload)

    if only:
        return
    # snapshot / resume golden on mixed3d (sim.py:187-220)
    rcfg = build(CASES["mixed3d"], rns)
    snap = rsim.snapshot_state(rcfg, None, 47)
    flat = {"step": np.int64(snap["step"]), "iterations": snap["iterations"]}
    for k, v in snap["fields"].items():
        flat["field__" + k] = v
    for key, v in snap["probes"].items():
        flat[_probe_key(key)] = v
    np.savez_compressed(OUT / "mixed3d_snapshot47.npz", **flat)
    print("snapshot golden written")

    # config loader parity on the shipped config
    from magphon.config import load_config as rload
    from paper_2510_22221_b200.config import load_config as mload
    path = "/root/reference/pkg/configs/cavity1d.cfg"
    a, b = rload(path), mload(path)
    assert (a.grid.cell_shape, a.grid.spacings) == (b.grid.cell_shape, b.grid.spacings) and a.cfl_factor == b.cfl_factor and a.t_end == b.t_end
    assert a.probes == b.probes and a.bias_sweep == b.bias_sweep
    assert a.source.__dict__ == b.source.__dict__ and a.boundaries.__dict__ == b.boundaries.__dict__
    assert a.llg_params.__dict__ == b.llg_params.__dict__ and a.bias_direction == b.bias_direction
    for f in ("sigma", "eps_r", "Ms", "alpha", "gamma_e", "Hbias"):
        assert np.array_equal(getattr(a.materials, f), getattr(b.materials, f)), f
    print("config loader parity ok")


if __name__ == "__main__":
    main()
