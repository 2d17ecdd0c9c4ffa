"""Damped-mode extraction for the acceptance tests (test utility).

A restatement of the subspace-rotation (ESPRIT) estimator the reference uses
to read modes off probe ringdowns (reference analysis.py:64-125): Hankel data
matrix of the samples, its dominant right-singular subspace, the least-squares
shift-invariance operator of that subspace, whose eigenvalues are the poles
z = exp((-r + 2 pi i f) dt); complex amplitudes by least squares on the first
<= 4096 samples.  Forward data matrix only (no forward-backward averaging,
which biases damped poles).  Post-processing is out of scope for the product
package; it lives here to check the CUDA path's probe series the way the
reference's acceptance suite checks its own.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Mode:
    freq: float
    amplitude: float      # |complex amplitude|
    decay_rate: float


def esprit(x, dt: float, order: int, columns: int = 1024) -> list[Mode]:
    x = np.asarray(x, dtype=float)
    n = x.size
    if n < 4 * order or columns <= order:
        raise ValueError("series too short for the requested order")
    hankel = np.lib.stride_tricks.sliding_window_view(x, columns)
    _, sv, vt = np.linalg.svd(hankel, full_matrices=False)
    if sv[order - 1] <= 1e-12 * sv[0]:
        raise ValueError("order exceeds the numerical rank of the data")
    basis = vt[:order].T
    rot = np.linalg.lstsq(basis[:-1], basis[1:], rcond=None)[0]
    poles = np.linalg.eigvals(rot)
    m = min(n, 4096)
    vander = poles[None, :] ** np.arange(m)[:, None]
    amps = np.linalg.lstsq(vander, x[:m], rcond=None)[0]
    out = []
    for z, a in zip(poles, amps):
        f = float(np.angle(z) / (2.0 * math.pi * dt))
        if f > 0:
            out.append(Mode(freq=f, amplitude=float(abs(a)),
                            decay_rate=float(-np.log(abs(z)) / dt)))
    return sorted(out, key=lambda md: md.freq)


def ringdown_modes(samples, dt: float) -> list[Mode]:
    """The acceptance suite's read-out of the cavity probe: ESPRIT(order 6,
    1024 columns) on the tail from sample 30000, decimated by 5, modes in
    10-18 GHz above 1e-7 of the drive amplitude."""
    samples = np.asarray(samples, dtype=float)
    tail = samples[30000:]
    modes = esprit(tail[::5], dt * 5, 6, 1024)
    drive = max(float(np.abs(samples).max()), 1.0)
    return [m for m in modes if 10e9 < m.freq < 18e9 and m.amplitude > 1e-7 * drive]


def strongest(modes, n: int):
    return sorted(sorted(modes, key=lambda m: -m.amplitude)[:n], key=lambda m: m.freq)
