"""fp32 field storage vs the fp64 reference: relative L2 errors per array.

    python tools/fp32_errors.py            (on a GPU box)

For every running golden case (reference outputs, tests/golden) and for C2/C3
from a mid-run state (vs the fp64 GPU path, itself bit-identical to the
oracle) prints rel-L2 of E, H, dM = M - M(t=0) and of the probe series."""
import json
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2510_22221_b200 import sim  # noqa: E402
from paper_2510_22221_b200.config import load_config  # noqa: E402
from paper_2510_22221_b200.grid import initial_magnetization  # noqa: E402
from tests.golden.cases import CASES, build, mirror_namespace  # noqa: E402
from tests.golden_io import load  # noqa: E402


def rel(a, b):
    nb = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / nb if nb > 0 else float(np.linalg.norm(a))


def errors(res, fields, probes, M0, its=None):
    st = res.lattice.state_arrays()
    out = {k: rel(st[k], v) for k, v in fields.items() if k != "M"}
    out["dM"] = rel(st["M"] - M0, fields["M"] - M0)
    out["probes"] = max((rel(res.probes[k].samples, v) for k, v in probes.items()), default=0.0)
    if its is not None and len(its):
        out["rstar_equal_frac"] = float(np.mean(res.iterations == its))
    return out


def main():
    rows = {}
    for name, case in CASES.items():
        if case.get("expect_failure"):
            continue
        g = load(name)
        cfg = build(case, mirror_namespace())
        res = sim.run(cfg, bias=case.get("bias"), storage="f32")
        mats = cfg.materials if case.get("bias") is None else sim._materials_with_bias(
            cfg.materials, case["bias"], cfg.bias_direction)
        rows[name] = errors(res, g["fields"], g["probes"], initial_magnetization(mats),
                            g["iterations"])
        print(name, json.dumps(rows[name]), flush=True)
    from tests.test_configs_gpu import mid_run_state
    for name, steps in (("c2", 50), ("c3", 50)):
        cfg = load_config(ROOT / "configs" / f"{name}.cfg")
        start = 200
        cfg = replace(cfg, t_end=(start + steps - 0.5) * cfg.dt)
        state = mid_run_state(cfg, 7)
        keys = [(p[0], (p[1], p[2], p[3])) for p in cfg.probes]
        snap = {"fields": state, "step": start, "probes": {k: np.zeros(start) for k in keys},
                "iterations": np.ones(start, dtype=int)}
        ref = sim.run(cfg, resume=snap)
        got = sim.run(cfg, resume=snap, storage="f32")
        rf = ref.lattice.state_arrays()
        rows[name] = errors(got, rf, {k: v.samples for k, v in ref.probes.items()},
                            state["M"], ref.iterations)
        print(name, json.dumps(rows[name]), flush=True)
    (ROOT / "gpurun_out").mkdir(exist_ok=True)
    (ROOT / "gpurun_out" / "fp32_errors.json").write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
