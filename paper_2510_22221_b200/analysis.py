"""Spectral post-processing needed by the sweep path.

Only the FFT magnitude spectrum that ``sweep`` emits (reference
``analysis.py:45-61``) lives here; ESPRIT and the other reference analysis
tools are host-side post-processing outside the hot path and accept this
package's ``ProbeSeries`` unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Spectrum:
    freqs: np.ndarray
    mags: np.ndarray
    meta: object = None

    def __post_init__(self) -> None:
        if len(self.freqs) != len(self.mags):
            raise ValueError("freqs and mags must have equal length")


def fft_magnitude(series, window: str = "none") -> Spectrum:
    """|rfft| of a uniformly sampled series on the grid k/(N dt).

    ``series``: a ProbeSeries (``samples``, ``dt_sample``) or a (samples, dt)
    pair; ``window``: "none" or "hann" (numpy's symmetric Hann).
    """
    if hasattr(series, "samples"):
        x, dt, meta = np.asarray(series.samples, float), float(series.dt_sample), series
    else:
        x, dt = np.asarray(series[0], float), float(series[1])
        meta = None
    if len(x) < 2:
        raise ValueError("need at least 2 samples")
    if window == "hann":
        x = x * np.hanning(len(x))
    elif window != "none":
        raise ValueError(f"unknown window {window!r}")
    return Spectrum(freqs=np.fft.rfftfreq(len(x), dt), mags=np.abs(np.fft.rfft(x)),
                    meta=meta)
