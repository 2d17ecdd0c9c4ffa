"""Per-cell material description (reference ``materials.py:19-99``).

The host keeps the dense per-cell arrays of the reference API because
callers build and inspect them; the device never sees them -- it gets a
uint8 material id per allocation entry plus a small coefficient table built
in :mod:`paper_2510_22221_b200.engine`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .constants import CONSTANTS


@dataclass(frozen=True)
class MaterialCell:
    sigma: float = 0.0
    eps_r: float = 1.0
    Ms: float = 0.0
    alpha: float = 0.0
    Hbias: tuple[float, float, float] = (0.0, 0.0, 0.0)
    gamma_e: float = CONSTANTS.gamma_e

    def __post_init__(self) -> None:
        checks = ((self.sigma >= 0, "sigma must be >= 0"),
                  (self.eps_r >= 1, "eps_r must be >= 1"),
                  (self.Ms >= 0, "Ms must be >= 0"),
                  (0.0 <= self.alpha <= 1.0, "alpha must be in [0,1]"))
        for ok, msg in checks:
            if not ok:
                raise ValueError(f"{msg} ({self})")

    @property
    def magnetic(self) -> bool:
        return self.Ms > 0.0


_ARRAYS = ("sigma", "eps_r", "Ms", "alpha", "gamma_e")


class MaterialMap:
    """Dense (nx, ny, nz) material arrays painted with half-open boxes."""

    def __init__(self, shape, background: MaterialCell | None = None):
        bg = background or MaterialCell()
        self.shape = tuple(int(s) for s in shape)
        if len(self.shape) != 3 or min(self.shape) < 1:
            raise ValueError(f"invalid cell counts {shape}")
        for name in _ARRAYS:
            setattr(self, name, np.full(self.shape, float(getattr(bg, name))))
        self.Hbias = np.empty((3,) + self.shape)
        self.Hbias[...] = np.asarray(bg.Hbias, float).reshape(3, 1, 1, 1)
        self._frozen = False

    def fill_box(self, cell: MaterialCell, i0: int = 0, i1: int | None = None,
                 j0: int = 0, j1: int | None = None, k0: int = 0,
                 k1: int | None = None) -> None:
        if self._frozen:
            raise RuntimeError("MaterialMap is frozen")
        lo = (i0, j0, k0)
        hi = tuple(n if h is None else h for h, n in zip((i1, j1, k1), self.shape))
        if not all(0 <= a <= b <= n for a, b, n in zip(lo, hi, self.shape)):
            raise ValueError(f"box ({i0}:{hi[0]},{j0}:{hi[1]},{k0}:{hi[2]}) "
                             f"outside grid {self.shape}")
        sl = tuple(slice(a, b) for a, b in zip(lo, hi))
        for name in _ARRAYS:
            getattr(self, name)[sl] = getattr(cell, name)
        for c in range(3):
            self.Hbias[(c,) + sl] = cell.Hbias[c]

    def freeze(self) -> "MaterialMap":
        for name in _ARRAYS + ("Hbias",):
            getattr(self, name).setflags(write=False)
        self._frozen = True
        return self

    @property
    def magnetic_mask(self) -> np.ndarray:
        return self.Ms > 0.0
