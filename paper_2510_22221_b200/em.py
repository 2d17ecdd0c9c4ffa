"""Electromagnetic run specification: source, walls, time step.

Host-side mirror of the spec types of reference ``em.py:33-101``.  The Yee
updates themselves (curl E, H, curl H, E, walls, source injection) run as
sm_100a kernels in ``csrc/``; nothing here touches field arrays.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .constants import CONSTANTS
from .grid import GridSpec

PEC = "PEC"
PMC = "PMC"
MUR1 = "MUR1"
CONDITIONS = (PEC, PMC, MUR1)
FACES = ("x0", "x1", "y0", "y1", "z0", "z1")


@dataclass(frozen=True)
class SourceSpec:
    """Modified-Gaussian soft source on one E entry (em.py:40-58)."""

    kind: str = "modified_gaussian"
    f0: float = 16e9
    Tp: float = 0.0625e-9
    amplitude: float = 1.0
    location: tuple[int, int, int] = (0, 0, 0)
    polarization: tuple[float, float, float] = (1.0, 0.0, 0.0)

    def __post_init__(self) -> None:
        if self.kind != "modified_gaussian":
            raise ValueError(f"unknown source kind {self.kind!r}")
        if not (self.f0 > 0 and self.Tp > 0):
            raise ValueError("f0 and Tp must be positive")
        norm = math.sqrt(sum(p * p for p in self.polarization))
        if not math.isclose(norm, 1.0, rel_tol=1e-9):
            raise ValueError("polarization must be a unit vector")


@dataclass(frozen=True)
class BoundarySpec:
    """Per-face wall condition, each one of PEC / PMC / MUR1 (em.py:61-79)."""

    x0: str = PEC
    x1: str = PEC
    y0: str = PEC
    y1: str = PEC
    z0: str = PEC
    z1: str = PEC

    def __post_init__(self) -> None:
        for face in FACES:
            cond = getattr(self, face)
            if cond not in CONDITIONS:
                raise ValueError(f"unknown boundary condition {cond!r} on {face}")

    @classmethod
    def uniform(cls, condition: str) -> "BoundarySpec":
        return cls(**dict.fromkeys(FACES, condition))


def cfl_timestep(spec: GridSpec, factor: float) -> float:
    """factor / (c0 sqrt(sum over active axes of 1/d^2)) -- em.py:82-93.

    Kept as the identical Python-float expression (``d**2``, Python ``sum``)
    so the host derives the same dt bit for bit.
    """
    if not 0 < factor <= 1:
        raise ValueError(f"CFL factor must be in (0,1], got {factor!r}")
    inv2 = sum(1.0 / d**2 for d, act in zip(spec.spacings, spec.active_axes) if act)
    if inv2 == 0.0:
        raise ValueError("grid has no active axis")
    return factor / (CONSTANTS.c0 * math.sqrt(inv2))


def source_value(src: SourceSpec, t: float) -> float:
    """amp * exp(-(t-3Tp)^2/(2Tp^2)) * cos(2 pi f0 t) -- em.py:96-101.

    Evaluated on the host with Python ``math`` (CUDA libm may differ by an
    ulp); the device receives the per-step values as an array.
    """
    if t < 0:
        raise ValueError("t must be >= 0")
    env = math.exp(-((t - 3.0 * src.Tp) ** 2) / (2.0 * src.Tp**2))
    return src.amplitude * env * math.cos(2.0 * math.pi * src.f0 * t)
