"""Host-side types of the coupled LLG fixed point.

The iteration itself runs on the GPU (``csrc/mpb_sweep.cuh`` ``k_llg_local``,
``csrc/mpb_kernels_split.cuh`` ``k_llg_fixup``); this module
keeps the reference's public types so callers catch the same exception
(reference ``pkg/src/magphon/llg.py:38-58``).
"""

from __future__ import annotations

from dataclasses import dataclass


class StepFailure(RuntimeError):
    """Per-step fixed point failed (diverging residual or budget exhausted).

    ``residual`` / ``iterations`` follow llg.py:139-148 exactly; ``step`` is
    attached by the run loop (sim.py:161-164).
    """

    def __init__(self, message: str, residual: float, iterations: int,
                 step: int | None = None):
        super().__init__(message)
        self.residual = residual
        self.iterations = iterations
        self.step = step


@dataclass(frozen=True)
class LlgIterationParams:
    tol: float = 1e-6
    max_iters: int = 50

    def __post_init__(self) -> None:
        if not self.tol > 0:
            raise ValueError("tol must be > 0")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
