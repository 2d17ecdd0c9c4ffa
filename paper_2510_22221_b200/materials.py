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
    """Dense (nx, ny, nz) material arrays painted with half-open boxes.

    The painting history (background + boxes in order) is kept, so a map can
    also be *lazy* (``lazy=True``): the dense float arrays of the reference
    API are only built if someone reads them, while the device path uses
    :meth:`painted` (one uint8 id per cell + the distinct cells) and
    :meth:`region` (an x-slab of the map) -- a 2048x2048x256 grid costs 1 GB
    of ids instead of 69 GB of per-cell doubles.
    """

    def __init__(self, shape, background: MaterialCell | None = None,
                 lazy: bool = False):
        bg = background or MaterialCell()
        self.shape = tuple(int(s) for s in shape)
        if len(self.shape) != 3 or min(self.shape) < 1:
            raise ValueError(f"invalid cell counts {shape}")
        self._bg = bg
        self._boxes: list = []
        self._frozen = False
        self.lazy = lazy
        if not lazy:
            self._materialize()

    # -- dense arrays (reference API) ------------------------------------------
    def _materialize(self) -> None:
        bg = self._bg
        for name in _ARRAYS:
            self.__dict__[name] = np.full(self.shape, float(getattr(bg, name)))
        hb = np.empty((3,) + self.shape)
        hb[...] = np.asarray(bg.Hbias, float).reshape(3, 1, 1, 1)
        self.__dict__["Hbias"] = hb
        for cell, sl in self._boxes:
            self._paint_dense(cell, sl)
        if self._frozen:
            for name in _ARRAYS + ("Hbias",):
                self.__dict__[name].setflags(write=False)

    def __getattr__(self, name):
        # only reached for attributes not yet set: the lazy dense arrays
        if name in _ARRAYS or name == "Hbias":
            if self.__dict__.get("_boxes") is None:
                raise AttributeError(name)
            self._materialize()
            return self.__dict__[name]
        raise AttributeError(name)

    @property
    def dense(self) -> bool:
        return "Ms" in self.__dict__

    def _paint_dense(self, cell, sl) -> None:
        for name in _ARRAYS:
            self.__dict__[name][sl] = getattr(cell, name)
        for c in range(3):
            self.__dict__["Hbias"][(c,) + sl] = cell.Hbias[c]

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
        self._boxes.append((cell, sl))
        if self.dense:
            self._paint_dense(cell, sl)

    def freeze(self) -> "MaterialMap":
        if self.dense:
            for name in _ARRAYS + ("Hbias",):
                getattr(self, name).setflags(write=False)
        self._frozen = True
        return self

    @property
    def magnetic_mask(self) -> np.ndarray:
        return self.Ms > 0.0

    # -- painted form (device path) ----------------------------------------------
    def cells(self) -> list:
        """Distinct cells, background first, in first-painted order."""
        out = [self._bg]
        for cell, _ in self._boxes:
            if cell not in out:
                out.append(cell)
        return out

    def painted(self):
        """(ids, cells): uint8 index into ``cells`` per cell, painted in
        box order (later boxes win, like fill_box)."""
        cells = self.cells()
        if len(cells) > 255:
            raise ValueError(f"{len(cells)} distinct materials in one map")
        index = {c: q for q, c in enumerate(cells)}
        ids = np.zeros(self.shape, dtype=np.uint8)
        for cell, sl in self._boxes:
            ids[sl] = index[cell]
        return ids, cells

    def magnetic_count(self) -> int:
        if self.dense:
            return int(np.count_nonzero(self.Ms > 0.0))
        ids, cells = self.painted()
        mag = np.array([c.magnetic for c in cells])
        return int(np.count_nonzero(mag[ids]))

    def region(self, c0: int, c1: int) -> "MaterialMap":
        """Lazy map of the cell planes [c0, c1) (boxes clipped and shifted)."""
        if not 0 <= c0 < c1 <= self.shape[0]:
            raise ValueError(f"region [{c0},{c1}) outside {self.shape[0]} planes")
        out = MaterialMap((c1 - c0,) + self.shape[1:], self._bg, lazy=True)
        for cell, sl in self._boxes:
            a, b = max(sl[0].start, c0), min(sl[0].stop, c1)
            if a < b:
                out._boxes.append((cell, (slice(a - c0, b - c0),) + sl[1:]))
        return out.freeze()

    def tiled_region(self, c0: int, c1: int) -> "MaterialMap":
        """Lazy map of the planes [c0, c1) of this map repeated along x
        (plane i is plane i mod nx) -- the weak-scaling slab of a line
        geometry that continues along x."""
        nx = self.shape[0]
        out = MaterialMap((c1 - c0,) + self.shape[1:], self._bg, lazy=True)
        for base in range((c0 // nx) * nx, c1, nx):      # copies do not overlap
            for cell, sl in self._boxes:
                a, b = max(sl[0].start + base, c0), min(sl[0].stop + base, c1)
                if a < b:
                    out._boxes.append((cell, (slice(a - c0, b - c0),) + sl[1:]))
        return out.freeze()

    def with_magnetic_bias(self, hbias) -> "MaterialMap":
        """Lazy copy whose magnetic cells carry ``hbias`` (3 floats)."""
        from dataclasses import replace
        hb = tuple(float(h) for h in hbias)
        swap = lambda c: replace(c, Hbias=hb) if c.magnetic else c   # noqa: E731
        out = MaterialMap(self.shape, swap(self._bg), lazy=True)
        out._boxes = [(swap(cell), sl) for cell, sl in self._boxes]
        return out.freeze()
