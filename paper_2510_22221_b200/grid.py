"""Yee-lattice geometry and the host copy of the field state.

Layout contract (reference ``grid.py:41-156``): each E/H component is a
C-order array of ``field_shape`` (n+1 along active axes, 1 along collapsed
ones); M is ``(3, nx, ny, nz)`` collocated with the same-index H entries.
On the device the same C order is kept with each x-plane padded to a
256-byte multiple ("Data layout in HBM").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .materials import MaterialMap

E_NAMES = ("Ex", "Ey", "Ez")
H_NAMES = ("Hx", "Hy", "Hz")
M_NAMES = ("Mx", "My", "Mz")


@dataclass(frozen=True)
class GridSpec:
    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float

    def __post_init__(self) -> None:
        for n in self.cell_shape:
            if not isinstance(n, int) or n < 1:
                raise ValueError(f"cell counts must be positive integers, got {n!r}")
        for d in self.spacings:
            if not d > 0:
                raise ValueError(f"cell sizes must be > 0, got {d!r}")

    @property
    def cell_shape(self) -> tuple[int, int, int]:
        return (self.nx, self.ny, self.nz)

    @property
    def field_shape(self) -> tuple[int, int, int]:
        return tuple(n + 1 if n > 1 else 1 for n in self.cell_shape)

    @property
    def active_axes(self) -> tuple[bool, bool, bool]:
        return tuple(n > 1 for n in self.cell_shape)

    @property
    def spacings(self) -> tuple[float, float, float]:
        return (self.dx, self.dy, self.dz)


class FieldLattice:
    """Host-side field state (what ``RunResult.lattice`` hands back)."""

    def __init__(self, spec: GridSpec, materials: MaterialMap):
        if tuple(materials.shape) != spec.cell_shape:
            raise ValueError(f"material map shape {materials.shape} does not "
                             f"match grid {spec.cell_shape}")
        self.spec = spec
        self.materials = materials
        for name in E_NAMES + H_NAMES:
            setattr(self, name, np.zeros(spec.field_shape))
        self.M = np.zeros((3,) + spec.cell_shape)

    @classmethod
    def adopt(cls, spec: GridSpec, materials, state: dict) -> "FieldLattice":
        """Lattice that takes ownership of freshly downloaded state arrays
        (no copy; same checks as load_state)."""
        lat = cls.__new__(cls)
        lat.spec = spec
        lat.materials = materials
        for name in E_NAMES + H_NAMES:
            a = state[name]
            if a.shape != spec.field_shape or a.dtype != np.float64:
                raise ValueError(f"snapshot shape mismatch for {name}")
            setattr(lat, name, a)
        if state["M"].shape != (3,) + spec.cell_shape:
            raise ValueError("snapshot shape mismatch for M")
        lat.M = state["M"]
        return lat

    def field(self, name: str) -> np.ndarray:
        if name in E_NAMES or name in H_NAMES:
            return getattr(self, name)
        if name in M_NAMES:
            return self.M[M_NAMES.index(name)]
        raise KeyError(f"unknown field component {name!r}")

    def sample(self, component: str, i: int, j: int, k: int) -> float:
        arr = self.field(component)
        if not all(0 <= x < n for x, n in zip((i, j, k), arr.shape)):
            raise IndexError(f"index ({i},{j},{k}) out of range for "
                             f"{component} with shape {arr.shape}")
        return float(arr[i, j, k])

    def state_arrays(self) -> dict[str, np.ndarray]:
        out = {name: getattr(self, name) for name in E_NAMES + H_NAMES}
        out["M"] = self.M
        return out

    def load_state(self, state: dict[str, np.ndarray]) -> None:
        for name in E_NAMES + H_NAMES + ("M",):
            dst = getattr(self, name)
            if np.shape(state[name]) != dst.shape:
                raise ValueError(f"snapshot shape mismatch for {name}")
        for name in E_NAMES + H_NAMES + ("M",):
            getattr(self, name)[...] = state[name]


def initial_magnetization(materials: MaterialMap) -> np.ndarray:
    """M = Ms * unit(Hbias) in magnetic cells, +x where the bias is zero,
    0 elsewhere (grid.py:140-156); computed on the host once per run."""
    if getattr(materials, "lazy", False):
        return _initial_magnetization_painted(materials)
    M = np.zeros((3,) + tuple(materials.shape))
    mag = materials.magnetic_mask
    if mag.any():
        hb = materials.Hbias[:, mag]
        norm = np.sqrt((hb * hb).sum(axis=0))
        unit = np.zeros_like(hb)
        has = norm > 0
        unit[:, has] = hb[:, has] / norm[has]
        unit[0, ~has] = 1.0
        M[:, mag] = materials.Ms[mag] * unit
    return M


def _initial_magnetization_painted(materials) -> np.ndarray:
    """initial_magnetization of a lazy map: the same per-cell expressions
    evaluated once per distinct cell, then scattered by material id."""
    ids, cells = materials.painted()
    nc = len(cells)
    M = np.zeros((3,) + tuple(materials.shape))
    if not any(c.Ms > 0.0 for c in cells):
        return M
    hb = np.array([c.Hbias for c in cells], dtype=float).T.reshape(3, nc)
    Ms = np.array([c.Ms for c in cells], dtype=float)
    mag = Ms > 0.0
    vec = np.zeros((3, nc))
    if mag.any():
        h = hb[:, mag]
        norm = np.sqrt((h * h).sum(axis=0))
        unit = np.zeros_like(h)
        has = norm > 0
        unit[:, has] = h[:, has] / norm[has]
        unit[0, ~has] = 1.0
        vec[:, mag] = Ms[mag] * unit
    # scatter into the magnetic cells only (a few % of the grid)
    where = np.flatnonzero(mag[ids])
    q = ids.reshape(-1)[where]
    for c in range(3):
        M[c].reshape(-1)[where] = vec[c][q]
    return M


def allocate(spec: GridSpec, materials: MaterialMap) -> FieldLattice:
    lat = FieldLattice(spec, materials)
    lat.M[...] = initial_magnetization(materials)
    return lat
