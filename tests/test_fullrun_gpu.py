"""The reference's only shipped run, full length, on the CUDA path.

``configs/cavity1d.cfg`` restates ``pkg/configs/cavity1d.cfg`` (the loader
parity is checked by the golden's generator).  3 ns = 499,655 coupled steps
through ``sim.run``; every probe sample, every LLG iteration count and the
final E/H/M arrays must be bit-identical to the reference's own full run,
recorded as SHA-256 digests in tests/golden/cavity1d_full.json
(tests/golden/make_fullrun_golden.py)."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from paper_2510_22221_b200 import sim
from paper_2510_22221_b200.config import load_config

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def digest(a) -> str:
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


# line kernel (default for z-lines) and the general kernels; either way the
# 499,655 steps cross eight 65,536-step host staging chunks of mpb_run
@pytest.mark.parametrize("line", ["1", "0"])
def test_shipped_cavity_full_length_bitwise(line, monkeypatch):
    monkeypatch.setenv("MPB_LINE", line)
    gold = json.loads((ROOT / "tests" / "golden" / "cavity1d_full.json").read_text())
    res = sim.run(load_config(ROOT / "configs" / "cavity1d.cfg"))
    assert res.steps == gold["steps"] == 499655
    for k, v in res.probes.items():
        name = f"{k[0]}_{k[1][0]}_{k[1][1]}_{k[1][2]}"
        assert float(np.abs(v.samples).max()) == gold["max_abs_probe"][name], name
        assert digest(v.samples) == gold["probes"][name], name
    its = np.asarray(res.iterations, dtype=np.int64)
    counts = {str(int(r)): int(c) for r, c in zip(*np.unique(its, return_counts=True))}
    assert counts == gold["r_star_counts"]
    assert digest(its) == gold["iterations"]
    for k, v in res.lattice.state_arrays().items():
        assert digest(v) == gold["fields"][k], k
