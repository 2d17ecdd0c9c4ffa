"""Spectral post-processing of probe series.

* ``fft_magnitude`` -- the Hann-window spectrum ``sweep`` emits (reference
  ``analysis.py:45-61``), on the host: numpy's pocketfft gives the
  reference's bits, and its 211 ms for the shipped 499,655-sample series is
  7% of the 3.0 s GPU run per bias and overlaps the other biases' runs.
* ``esprit`` -- the subspace mode extraction (reference ``analysis.py:64-125``)
  with its Hankel products on the GPU: the reference's
  full SVD takes longer than the simulation it post-processes.
The other reference analysis tools accept this package's ``ProbeSeries``.
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


# ---------------------------------------------------------------------------
# Subspace (ESPRIT) mode extraction with the Hankel products on the GPU
# (reference analysis.py:64-125)
# ---------------------------------------------------------------------------

Q_CAP = 1e9                       # analysis.py:15


@dataclass(frozen=True)
class ModeEstimate:               # analysis.py:30-37
    freq: float
    Q: float
    amplitude: complex
    decay_rate: float
    q_capped: bool = False
    growing: bool = False


def _hankel_mul(x, columns, block, transpose, device):
    """X @ block (transpose=0) or X^T @ block (transpose=1) on the GPU,
    X[t][a] = x[t + a] (mpb_hankel_mul)."""
    import ctypes as C

    from . import _native as N
    x = np.ascontiguousarray(x, dtype=np.float64)
    block = np.ascontiguousarray(block, dtype=np.float64)
    m = x.size - columns + 1
    r = block.shape[1]
    out = np.empty(((columns if transpose else m), r))
    P = C.POINTER(C.c_double)
    N.check(N.load_library().mpb_hankel_mul(
        device, x.ctypes.data_as(P), x.size, columns, r, int(transpose),
        block.ctypes.data_as(P), out.ctypes.data_as(P)))
    return out


def esprit(series, model_order: int, hankel_columns: int | None = None, *,
           device: int = 0, oversample: int = 12, power: int = 3,
           seed: int = 20251022) -> list:
    """Damped-sinusoid modes by rotational invariance -- the reference's
    ``analysis.esprit`` (analysis.py:64-115: forward Hankel data matrix,
    dominant right-singular subspace, least-squares shift invariance,
    eigenvalues -> f, decay rate, Q; amplitudes by Vandermonde least
    squares), with the same arguments, errors and ModeEstimate output.

    The reference takes the full SVD of the (N - L + 1) x L Hankel matrix on
    the host (~2.4 s for the acceptance suite's 14,000 x 1024 ringdowns).
    Here the dominant subspace comes from a randomized range finder whose
    O(N L r) products with X run on the GPU (mpb_hankel_mul, r = order +
    ``oversample`` <= 32 probe vectors, ``power`` subspace iterations with
    Householder re-orthonormalisation); the r x L projection, the K x K
    shift solve, the eigenvalues and the amplitudes are small host algebra
    exactly as in the reference.  The subspace, hence every pole, agrees
    with the full SVD to rounding whenever the retained modes stand above
    the rest of the spectrum (tests/test_esprit_gpu.py); a fixed seed keeps
    the result deterministic.
    """
    if hasattr(series, "samples"):
        x, dt = np.asarray(series.samples, float), float(series.dt_sample)
    else:
        x, dt = np.asarray(series[0], float), float(series[1])
    n = len(x)
    if n < 4 * model_order:
        raise ValueError(f"series length {n} < 4*model_order")
    L = hankel_columns or min(n // 3, 1024)
    if L <= model_order:
        raise ValueError("hankel_columns must exceed model_order")
    m = n - L + 1
    r = int(min(model_order + oversample, 32, L, m))
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(_hankel_mul(x, L, rng.standard_normal((L, r)), 0, device))
    for _ in range(power):
        z, _ = np.linalg.qr(_hankel_mul(x, L, q, 1, device))
        q, _ = np.linalg.qr(_hankel_mul(x, L, z, 0, device))
    b = _hankel_mul(x, L, q, 1, device).T            # Q^T X, r x L
    _, s, vt = np.linalg.svd(b, full_matrices=False)
    if s[model_order - 1] <= 1e-12 * s[0]:
        raise ValueError(
            f"model order {model_order} exceeds numerical rank of the data "
            f"(singular value ratio {s[model_order - 1] / s[0]:.2e})")
    V = vt[:model_order].T
    phi = np.linalg.lstsq(V[:-1], V[1:], rcond=None)[0]
    lam = np.linalg.eigvals(phi)
    nn = np.arange(n)
    mm = min(n, 4096)
    amp = np.linalg.lstsq(lam[None, :] ** nn[:mm, None], x[:mm], rcond=None)[0]
    modes = []
    for lv, av in zip(lam, amp):
        f = float(np.angle(lv) / (2.0 * np.pi * dt))
        if f <= 0:
            continue
        rr = float(-np.log(np.abs(lv)) / dt)
        growing = np.abs(lv) > 1.0 + 1e-9
        if rr > 0:
            qq = np.pi * f / rr
            capped = qq > Q_CAP
        else:
            qq, capped = Q_CAP, True
        modes.append(ModeEstimate(freq=f, Q=min(qq, Q_CAP), amplitude=av, decay_rate=rr,
                                  q_capped=capped, growing=bool(growing)))
    modes.sort(key=lambda md: md.freq)
    return modes
