"""Load the committed golden fixtures (tests/golden/*.npz)."""

from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    data = np.load(GOLDEN / f"{name}.npz")
    out = {"fields": {}, "probes": {}}
    for k in data.files:
        if k.startswith("field__"):
            out["fields"][k[7:]] = data[k]
        elif k.startswith("probe__"):
            comp, i, j, kk = k[7:].split("__")
            out["probes"][(comp, (int(i), int(j), int(kk)))] = data[k]
        else:
            out[k] = data[k]
    return out
