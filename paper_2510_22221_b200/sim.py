"""Run orchestration -- the drop-in for reference ``magphon.sim``.

``run(config, bias=None, resume=None) -> RunResult`` keeps the reference
signature, return type, error behaviour and bit-for-bit results
(reference sim.py:125-180); the time loop itself executes on the B200
through the C ABI (``engine.DeviceRun``).  Snapshot/restart
(sim.py:187-220) and bias sweeps (sim.py:243-260) are mirrored on top.

Host work per run: material table + initial M (numpy, once), the per-step
source values v((n+1) dt) (Python ``math``, once per step -- they must be the
reference's exact doubles), and the final state download.
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace

import functools

import numpy as np

from . import em, llg
from .engine import DeviceRun
from .grid import FieldLattice, GridSpec, initial_magnetization
from .materials import MaterialMap

_FIELD_NAMES = ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")
_VALID_COMPS = _FIELD_NAMES + ("Mx", "My", "Mz")


@dataclass(frozen=True)
class SimConfig:
    grid: GridSpec
    materials: MaterialMap
    source: em.SourceSpec
    boundaries: em.BoundarySpec
    cfl_factor: float
    t_end: float
    probes: tuple[tuple[str, int, int, int], ...]
    bias_sweep: tuple[float, ...] = ()
    bias_direction: tuple[float, float, float] = (1.0, 0.0, 0.0)
    llg_params: llg.LlgIterationParams = field(default_factory=llg.LlgIterationParams)
    spectrum_probe: int = 0

    def __post_init__(self) -> None:
        if not self.t_end > 0:
            raise ValueError("t_end must be > 0")
        for comp, i, j, k in self.probes:
            lim = self.grid.cell_shape if comp.startswith("M") else self.grid.field_shape
            if not all(0 <= x < n for x, n in zip((i, j, k), lim)):
                raise ValueError(f"probe {(comp, i, j, k)} outside grid")

    @property
    def dt(self) -> float:
        return em.cfl_timestep(self.grid, self.cfl_factor)

    @property
    def n_steps(self) -> int:
        return int(np.ceil(self.t_end / self.dt))


@dataclass
class ProbeSeries:
    component: str
    location: tuple[int, int, int]
    bias: float
    dt_sample: float
    samples: np.ndarray

    def __len__(self) -> int:
        return len(self.samples)


@dataclass
class RunResult:
    probes: dict
    lattice: FieldLattice
    iterations: np.ndarray
    steps: int
    bias: float


def _materials_with_bias(materials, bias: float, direction) -> MaterialMap:
    """Copy with the magnetic cells' bias replaced (sim.py:82-97)."""
    if getattr(materials, "lazy", False):
        unit = np.asarray(direction, float)
        unit = unit / np.linalg.norm(unit)
        return materials.with_magnetic_bias([bias * unit[c] for c in range(3)])
    out = MaterialMap(materials.shape)
    for name in ("sigma", "eps_r", "Ms", "alpha", "gamma_e", "Hbias"):
        setattr(out, name, np.array(getattr(materials, name), copy=True))
    mag = out.Ms > 0
    unit = np.asarray(direction, float)
    unit = unit / np.linalg.norm(unit)
    for c in range(3):
        out.Hbias[c][mag] = bias * unit[c]
    return out.freeze()


def _wrap_source(loc, shape):
    out = []
    for x, n in zip(loc, shape):
        if not -n <= x < n:
            raise IndexError(f"source index {tuple(loc)} out of bounds for "
                             f"field shape {shape}")
        out.append(x % n)
    return tuple(out)


@functools.lru_cache(maxsize=16)
def _source_values(src: em.SourceSpec, dt: float, start: int, stop: int) -> np.ndarray:
    return np.array([em.source_value(src, (n + 1) * dt) for n in range(start, stop)],
                    dtype=np.float64)


def source_values(src: em.SourceSpec, dt: float, start: int, stop: int) -> np.ndarray:
    """v((n+1) dt) for n in [start, stop) with the reference's Python math
    (one Python call per step, so cached: the runs of a bias sweep share it)."""
    return _source_values(src, float(dt), int(start), int(stop)).copy()


def _device_run_args(config, keys) -> dict:
    """Validate probes/walls/source like the reference would at run time and
    return the device-facing source and wall arguments.

    The reference raises these errors inside its first step, in this order:
    MUR1 on a collapsed axis (``em._capture_mur_planes``, em.py:306-321),
    the source index (``inject_soft_source``), then each probe in config
    order (``FieldLattice.sample``: unknown component, then index range).
    """
    fs = config.grid.field_shape
    b = config.boundaries
    for face, axis in (("x0", 0), ("x1", 0), ("y0", 1), ("y1", 1), ("z0", 2), ("z1", 2)):
        if getattr(b, face) == em.MUR1 and not config.grid.active_axes[axis]:
            raise ValueError(f"MUR1 on collapsed axis face {face}")
    pol = config.source.polarization
    loc = config.source.location
    if any(p != 0.0 for p in pol):
        loc = _wrap_source(loc, fs)
    else:
        loc = (0, 0, 0)
    for comp, (i, j, k) in keys:
        if comp not in _VALID_COMPS:
            raise KeyError(f"unknown field component {comp!r}")
        lim = config.grid.cell_shape if comp.startswith("M") else fs
        if not all(0 <= x < n for x, n in zip((i, j, k), lim)):
            raise IndexError(f"index ({i},{j},{k}) out of range for {comp}")
    return {"source_loc": loc, "source_pol": pol, "boundaries": b}


def _unchecked_run_args(config) -> dict:
    """Device arguments that skip the run-time checks: no source, and PEC in
    place of MUR1 on collapsed axes.  Used only where the reference would
    not reach those checks (no step to run) or to find out whether the LLG
    of the first step fails before them."""
    b = config.boundaries
    repl = {face: em.PEC for face, axis in (("x0", 0), ("x1", 0), ("y0", 1), ("y1", 1),
                                            ("z0", 2), ("z1", 2))
            if getattr(b, face) == em.MUR1 and not config.grid.active_axes[axis]}
    return {"source_loc": (0, 0, 0), "source_pol": (0.0, 0.0, 0.0),
            "boundaries": replace(b, **repl) if repl else b}


def _device_run(config, materials, keys, device: int = 0, *, checked: bool = True,
                **kw) -> DeviceRun:
    a = _device_run_args(config, keys) if checked else _unchecked_run_args(config)
    return DeviceRun(config.grid, materials, a["boundaries"], a["source_loc"],
                     a["source_pol"], keys if checked else [], config.llg_params,
                     config.dt, device=device, **kw)


def _raise_failure(fail, config):
    step, res, it, kind = fail
    if kind == 1:
        msg = (f"fixed-point iteration diverging (residual {res:.3e} "
               f"after {it} iterates)")
    elif kind == 4:   # only from mpb_run_device (mpb_run continues the step)
        msg = (f"multi-rank step suspended: global residual back above tol at "
               f"iterate {it} (residual {res:.3e}); continue it through mpb_run")
    else:
        msg = (f"fixed-point iteration did not reach tol "
               f"{config.llg_params.tol:.1e} in "
               f"{config.llg_params.max_iters} iterates (residual {res:.3e})")
    raise llg.StepFailure(msg, res, it, step=step)


def run(config: SimConfig, bias: float | None = None, resume: dict | None = None,
        *, device: int = 0, kernel_variant: int = 0, storage: str = "f64",
        _final_state: bool = True) -> RunResult:
    """Execute a full run on the GPU (reference sim.py:125-180).

    With ``bias`` the magnets' bias is overridden along
    ``config.bias_direction``; ``resume`` continues from a snapshot dict and
    is bit-identical to an uninterrupted run.  ``storage="f32"`` (not in the
    reference API) keeps E and H in fp32 on the device -- half the HBM
    traffic per step, M and the LLG still fp64 -- and agrees with the fp64
    path within the tolerance tests/test_fp32_gpu.py states, not bitwise.
    """
    materials = config.materials if bias is None else _materials_with_bias(
        config.materials, bias, config.bias_direction)
    dt = config.dt
    n_steps = config.n_steps
    buffers = {(p[0], (p[1], p[2], p[3])): [] for p in config.probes}
    iters_prefix: list = []
    start = 0
    if resume is not None:
        start = int(resume["step"])
        for key, vals in resume["probes"].items():
            buffers[key] = list(vals)
        iters_prefix = list(resume["iterations"])
    keys = list(buffers)
    count = max(0, n_steps - start)
    pending = None
    try:
        _device_run_args(config, keys)
    except (ValueError, IndexError, KeyError) as exc:
        # the reference raises these inside its first step, after that
        # step's LLG; with no step left to run it never reaches them
        pending = exc
    dev = _device_run(config, materials, keys, device=device, checked=pending is None,
                      kernel_variant=kernel_variant, storage=storage)
    try:
        if resume is not None:
            st = resume["fields"]
            dev.load_state({n: st[n] for n in _FIELD_NAMES}, st["M"])
        else:
            dev.load_state(None, initial_magnetization(materials))   # E = H = 0
        if pending is not None and count > 0:
            # one step of the unchecked run: a StepFailure of the first
            # step's LLG wins over the error its E update would raise
            _, _, fail = dev.run(start, np.zeros(1))
            if fail is not None:
                _raise_failure(fail, config)
            raise pending
        vals = source_values(config.source, dt, start, n_steps)
        probe_rows, iters, fail = dev.run(start, vals)
        if fail is not None:
            _raise_failure(fail, config)
        # (a bias sweep keeps only the probes: no final-state download)
        state = dev.save_state() if _final_state else None
    finally:
        dev.close()
    lat = FieldLattice.adopt(config.grid, materials, state) if state is not None else None
    b = 0.0 if bias is None else bias
    probes = {}
    for p, key in enumerate(keys):
        tail = probe_rows[:count, p] if count else np.zeros(0)
        samples = np.concatenate([np.asarray(buffers[key], dtype=np.float64), tail])
        probes[key] = ProbeSeries(component=key[0], location=key[1], bias=b,
                                  dt_sample=dt, samples=samples)
    if dev.n_magnetic > 0:
        iterations = np.asarray(iters_prefix + list(iters[:count]), dtype=int)
    else:
        iterations = np.asarray(iters_prefix, dtype=int)
    return RunResult(probes=probes, lattice=lat, iterations=iterations,
                     steps=n_steps, bias=b)


# ---------------------------------------------------------------------------
# snapshot / restart (sim.py:187-220)
# ---------------------------------------------------------------------------

def snapshot_state(config: SimConfig, bias: float | None, until_step: int) -> dict:
    res = run(replace(config, t_end=until_step * config.dt), bias=bias)
    return {"fields": res.lattice.state_arrays(), "step": res.steps,
            "probes": {k: v.samples for k, v in res.probes.items()},
            "iterations": res.iterations}


def save_snapshot(path, snap: dict) -> None:
    flat = {f"field_{k}": v for k, v in snap["fields"].items()}
    flat["step"] = np.asarray(snap["step"])
    flat["iterations"] = np.asarray(snap["iterations"])
    for (comp, loc), vals in snap["probes"].items():
        flat["probe_{}_{}_{}_{}".format(comp, *loc)] = np.asarray(vals)
    np.savez(path, **flat)


def load_snapshot(path) -> dict:
    data = np.load(path)
    fields, probes = {}, {}
    for key in data.files:
        if key.startswith("field_"):
            fields[key[6:]] = data[key]
        elif key.startswith("probe_"):
            comp, i, j, k = key[6:].rsplit("_", 3)
            probes[(comp, (int(i), int(j), int(k)))] = data[key]
    return {"fields": fields, "step": int(data["step"]), "probes": probes,
            "iterations": data["iterations"]}


# ---------------------------------------------------------------------------
# bias sweep (sim.py:227-260): one run per bias, replicas across GPUs
# ---------------------------------------------------------------------------

@dataclass
class SpectrumMap:
    biases: np.ndarray
    freqs: np.ndarray
    mags: np.ndarray


def _sweep_one(args):
    config, bias, device = args
    from .analysis import fft_magnitude
    res = run(config, bias=bias, device=device, _final_state=False)
    probe = list(res.probes.values())[config.spectrum_probe]
    spec = fft_magnitude(probe, window="hann")
    return spec.freqs, spec.mags


def _sweep_device(args):
    """All biases assigned to one GPU, ``streams`` of them at a time: each run
    owns a handle with its own CUDA stream, driven from its own host thread
    (the C ABI releases the GIL), so small grids that cannot fill a B200 on
    their own share it."""
    jobs, streams = args
    if streams <= 1 or len(jobs) <= 1:
        return [_sweep_one(j) for j in jobs]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=streams) as ex:
        return list(ex.map(_sweep_one, jobs))


def _gpu_count() -> int:
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def sweep(config: SimConfig, biases=None, parallel: int = 1) -> SpectrumMap:
    """Hann-window FFT magnitude of the spectrum probe for every bias.

    ``parallel > 1`` runs up to ``parallel`` biases at once: spread over the
    GPUs (one spawned process per GPU, never forked after CUDA init) and, when
    ``parallel`` exceeds the GPU count, several concurrent runs per GPU on
    separate streams.  Every run is independent and deterministic, and rows
    are assembled in bias order, so serial and parallel sweeps are identical
    (reference sim.py:243-260).
    """
    biases = np.asarray(config.bias_sweep if biases is None else biases, float)
    if biases.size == 0:
        raise ValueError("bias sweep must be non-empty")
    ngpu = max(1, _gpu_count())
    parallel = max(1, min(int(parallel), biases.size))
    gpus = min(parallel, ngpu)
    streams = -(-parallel // gpus)                       # concurrent runs per GPU
    per_gpu = [[] for _ in range(gpus)]
    order = []
    for i, b in enumerate(biases):
        per_gpu[i % gpus].append((config, float(b), i % gpus))
        order.append((i % gpus, len(per_gpu[i % gpus]) - 1))
    if gpus > 1:
        import multiprocessing as mp
        with mp.get_context("spawn").Pool(gpus) as pool:
            done = pool.map(_sweep_device, [(jobs, streams) for jobs in per_gpu])
    else:
        done = [_sweep_device((per_gpu[0], streams))]
    rows = [done[g][q] for g, q in order]
    return SpectrumMap(biases=biases, freqs=rows[0][0], mags=np.stack([r[1] for r in rows]))
