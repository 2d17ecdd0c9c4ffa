"""SI constants and Gaussian-unit conversions used at the config boundary.

Mirrors ``magphon.constants`` (reference ``pkg/src/magphon/constants.py:18-66``);
the numeric values must be the identical Python doubles because every
kernel coefficient is derived from them on the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

_4PI = 4.0 * math.pi


@dataclass(frozen=True)
class PhysicalConstants:
    eps0: float = 8.8541878128e-12   # F/m
    mu0: float = 4e-7 * math.pi      # H/m
    c0: float = 299792458.0          # m/s
    gamma_e: float = -1.759e11       # C/kg, electron (negative)

    @property
    def gamma_eff(self) -> float:
        return self.mu0 * abs(self.gamma_e)


CONSTANTS = PhysicalConstants()


def _finite(v: float) -> float:
    if not math.isfinite(v):
        raise ValueError(f"non-finite field value: {v!r}")
    return v


def oersted_to_si(h: float) -> float:
    """Oe -> A/m (1 Oe = 1000/(4 pi) A/m); constants.py:36-43."""
    return _finite(h) * 1000.0 / _4PI


def si_to_oersted(h: float) -> float:
    return _finite(h) * _4PI / 1000.0


def gauss_4piMs_to_si(b: float) -> float:
    """4 pi Ms in Gauss -> Ms in A/m; constants.py:53-66."""
    if b < 0:
        raise ValueError(f"4*pi*Ms must be non-negative, got {b!r}")
    return b * 1000.0 / _4PI
