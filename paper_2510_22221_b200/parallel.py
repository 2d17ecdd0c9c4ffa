"""x-slab decomposition across GPUs -- host logic.

One process per GPU (``torchrun``); ``torch.distributed`` carries the
plumbing (rendezvous, NCCL unique id, result gathering) and the C library
does the per-step halo exchange and LLG all-reduce over NCCL itself.

Partition: rank r owns cell planes ``[x_lo, x_hi)`` (balanced, >= 2 planes
each); the last rank also owns field plane nx.  Each rank keeps one ghost
field plane on each side: field planes ``[max(0, x_lo-1), min(F, x_hi'+1))``
with ``x_hi' = F`` on the last rank; cell (material, M) planes
``[max(0, x_lo-1), min(nx, x_hi+1))``.  The same functions drive the
per-process host tests in ``tests/test_parallel_host.py`` (gloo, 2 ranks) and
the one-GPU rank emulation in ``tests/test_slab_gpu.py``, which checks the
plan bit for bit against the single-domain oracle goldens.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def partition(nx: int, nranks: int) -> list[tuple[int, int]]:
    """Balanced contiguous cell-plane ranges, >= 2 planes per rank."""
    if nranks < 1 or nx < 2 * nranks:
        raise ValueError(f"cannot split {nx} cell planes over {nranks} ranks "
                         f"(need >= 2 planes per rank)")
    base, extra = divmod(nx, nranks)
    out, lo = [], 0
    for r in range(nranks):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


@dataclass(frozen=True)
class Slab:
    nranks: int
    rank: int
    nx: int               # global cell count along x
    x_lo: int             # owned cell planes [x_lo, x_hi)
    x_hi: int
    any_magnetic: bool = False
    nccl_id: bytes = bytes(128)

    @property
    def F(self) -> int:
        return self.nx + 1 if self.nx > 1 else 1

    @property
    def owned_fields(self) -> tuple[int, int]:
        """Owned field planes (global), [c0, c1)."""
        return self.x_lo, (self.F if self.x_hi == self.nx else self.x_hi)

    @property
    def field_range(self) -> tuple[int, int]:
        """Field planes held locally (owned + ghosts)."""
        c0, c1 = self.owned_fields
        return max(0, c0 - 1), min(self.F, c1 + 1)

    @property
    def cell_range(self) -> tuple[int, int]:
        return max(0, self.x_lo - 1), min(self.nx, self.x_hi + 1)


def make_slabs(nx: int, nranks: int, any_magnetic: bool = False) -> list[Slab]:
    return [Slab(nranks, r, nx, lo, hi, any_magnetic)
            for r, (lo, hi) in enumerate(partition(nx, nranks))]


def local_fields(slab: Slab, global_arr: np.ndarray) -> np.ndarray:
    f0, f1 = slab.field_range
    return np.ascontiguousarray(global_arr[f0:f1])


def local_cells(slab: Slab, global_arr: np.ndarray, axis: int = 0) -> np.ndarray:
    c0, c1 = slab.cell_range
    sl = [slice(None)] * global_arr.ndim
    sl[axis] = slice(c0, c1)
    return np.ascontiguousarray(global_arr[tuple(sl)])


def owned_part(slab: Slab, local_arr: np.ndarray) -> np.ndarray:
    """Owned field planes of a local (ghosted) array."""
    f0, _ = slab.field_range
    c0, c1 = slab.owned_fields
    return local_arr[c0 - f0:c1 - f0]


def owned_cells(slab: Slab, local_m: np.ndarray) -> np.ndarray:
    c0, _ = slab.cell_range
    return local_m[:, slab.x_lo - c0:slab.x_hi - c0]


def nccl_unique_id(dist) -> bytes:
    """Rank 0 creates the NCCL id, every rank receives it (torch.distributed)."""
    from . import _native as N
    import ctypes as C
    buf = [None]
    if dist.get_rank() == 0:
        raw = (C.c_uint8 * 128)()
        N.check(N.load_library().mpb_nccl_unique_id(raw))
        buf[0] = bytes(raw)
    dist.broadcast_object_list(buf, src=0)
    return buf[0]


# ---------------------------------------------------------------------------
# Material slices and the in-process group (one GPU, emulated ranks)
# ---------------------------------------------------------------------------

class _MaterialSlab:
    """Cell-plane slice of a MaterialMap (what DeviceRun needs)."""

    def __new__(cls, materials, slab: Slab):
        if getattr(materials, "lazy", False):      # painted map: slice the boxes
            return materials.region(*slab.cell_range)
        return super().__new__(cls)

    def __init__(self, materials, slab: Slab):
        c0, c1 = slab.cell_range
        for name in ("sigma", "eps_r", "Ms", "alpha", "gamma_e"):
            setattr(self, name, np.asarray(getattr(materials, name))[c0:c1])
        self.Hbias = np.asarray(materials.Hbias)[:, c0:c1]
        self.shape = self.Ms.shape

    @property
    def magnetic_mask(self):
        return self.Ms > 0.0


def slab_device_runs(config, materials, keys, slabs, device=0, **kw):
    """One DeviceRun per slab (all on ``device``; no NCCL when the slabs'
    nccl_id is zero -> usable with mpb_group_run)."""
    from .sim import _device_run_args
    from .engine import DeviceRun
    args = _device_run_args(config, keys)
    runs = []
    for sl in slabs:
        runs.append(DeviceRun(config.grid, _MaterialSlab(materials, sl), args["boundaries"],
                              args["source_loc"], args["source_pol"], keys,
                              config.llg_params, config.dt, device=device, slab=sl, **kw))
    return runs


def run_group(config, nranks: int, bias=None, device: int = 0, state=None, start: int = 0,
              stats: dict | None = None):
    """Run ``config`` as an ``nranks``-slab decomposition emulated on one GPU
    (mpb_group_run).  Returns (fields dict, M, probes dict, iterations) in
    the global layout -- must equal sim.run bit for bit.  ``state`` (global
    E/H fields and M) with ``start`` continues from a mid-run state; the
    probes and iterations returned then cover steps [start, n_steps)."""
    import ctypes as C

    from . import _native as N
    from .grid import initial_magnetization
    from .sim import _materials_with_bias, source_values
    materials = config.materials if bias is None else _materials_with_bias(
        config.materials, bias, config.bias_direction)
    keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in config.probes))
    any_mag = bool(np.count_nonzero(np.asarray(materials.Ms) > 0))
    slabs = make_slabs(config.grid.nx, nranks, any_mag)
    runs = slab_device_runs(config, materials, keys, slabs, device=device)
    try:
        fs = config.grid.field_shape
        names = ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")
        if state is None:
            zeros = np.zeros(fs)
            state = dict({n: zeros for n in names}, M=initial_magnetization(materials))
        for r, sl in zip(runs, slabs):
            r.load_state({n: local_fields(sl, state[n]) for n in names},
                         local_cells(sl, state["M"], axis=1))
        steps = config.n_steps - start
        src = source_values(config.source, config.dt, start, config.n_steps)
        probes = [np.zeros((steps, max(1, len(keys)))) for _ in runs]
        iters = np.zeros(steps, dtype=np.int32)
        hs = (C.c_void_p * nranks)(*[r.h for r in runs])
        pp = (C.POINTER(C.c_double) * nranks)(
            *[p.ctypes.data_as(C.POINTER(C.c_double)) for p in probes])
        fail = N.Failure()
        code = N.load_library().mpb_group_run(
            hs, nranks, start, steps, src.ctypes.data_as(C.POINTER(C.c_double)), pp,
            iters.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(fail))
        if code == N.ESTEP:
            return None, None, None, (int(fail.step), float(fail.residual),
                                      int(fail.iterations), int(fail.kind))
        N.check(code)
        if stats is not None:
            stats["continued_steps"] = int(N.load_library().mpb_continued_steps(runs[0].h))
        fields = {n: np.empty(fs) for n in ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")}
        M = np.empty((3,) + config.grid.cell_shape)
        for r, sl in zip(runs, slabs):
            st = r.save_state()
            c0, c1 = sl.owned_fields
            for n in fields:
                fields[n][c0:c1] = owned_part(sl, st[n])
            M[:, sl.x_lo:sl.x_hi] = owned_cells(sl, st["M"])
        out_probes = {}
        for p, (comp, loc) in enumerate(keys):
            owner = next(q for q, sl in enumerate(slabs)
                         if sl.owned_fields[0] <= loc[0] < sl.owned_fields[1])
            out_probes[(comp, loc)] = probes[owner][:, p].copy()
        its = iters.astype(int) if any_mag else np.zeros(0, dtype=int)
        return fields, M, out_probes, its
    finally:
        for r in runs:
            r.close()


# ---------------------------------------------------------------------------
# One process per GPU (torchrun): the NCCL data plane
# ---------------------------------------------------------------------------

def run_ranks(config, bias=None, state=None, start: int = 0):
    """Run ``config`` as an x-slab decomposition over the ranks of the
    initialised ``torch.distributed`` process group, one GPU per rank
    (``LOCAL_RANK``), the halo exchange and LLG all-reduces over NCCL inside
    the library (mpb_run).  The same contract as :func:`run_group`: on rank 0
    returns (fields, M, probes, iterations) in the global layout -- equal to
    sim.run bit for bit -- or (None, None, None, failure); other ranks return
    None."""
    import os
    from dataclasses import replace

    import torch.distributed as dist

    from .grid import initial_magnetization
    from .sim import _materials_with_bias, source_values
    world, rank = dist.get_world_size(), dist.get_rank()
    device = int(os.environ.get("LOCAL_RANK", rank))
    materials = config.materials if bias is None else _materials_with_bias(
        config.materials, bias, config.bias_direction)
    keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in config.probes))
    any_mag = bool(np.count_nonzero(np.asarray(materials.Ms) > 0))
    nccl_id = nccl_unique_id(dist)
    sl = replace(make_slabs(config.grid.nx, world, any_mag)[rank], nccl_id=nccl_id)
    run = slab_device_runs(config, materials, keys, [sl], device=device)[0]
    try:
        fs = config.grid.field_shape
        names = ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")
        if state is None:
            zeros = np.zeros(fs)
            state = dict({n: zeros for n in names}, M=initial_magnetization(materials))
        run.load_state({n: local_fields(sl, state[n]) for n in names},
                       local_cells(sl, state["M"], axis=1))
        probes, iters, fail = run.run(start, source_values(config.source, config.dt, start,
                                                           config.n_steps))
        if fail is not None:
            part = None
        else:
            st = run.save_state()
            part = {n: owned_part(sl, st[n]) for n in names}
            part["M"] = owned_cells(sl, st["M"])
            part["probes"] = probes
        parts = [None] * world if rank == 0 else None
        dist.gather_object((sl, part, fail), parts, dst=0)
    finally:
        run.close()
    if rank != 0:
        return None
    fails = [f for _, _, f in parts if f is not None]
    if fails:
        return None, None, None, fails[0]
    fields = {n: np.empty(fs) for n in names}
    M = np.empty((3,) + config.grid.cell_shape)
    for s, p, _ in parts:
        c0, c1 = s.owned_fields
        for n in names:
            fields[n][c0:c1] = p[n]
        M[:, s.x_lo:s.x_hi] = p["M"]
    out_probes = {}
    for q, (comp, loc) in enumerate(keys):
        s, p, _ = next(x for x in parts if x[0].owned_fields[0] <= loc[0] < x[0].owned_fields[1])
        out_probes[(comp, loc)] = p["probes"][:, q].copy()
    its = np.asarray(iters, dtype=int) if any_mag else np.zeros(0, dtype=int)
    return fields, M, out_probes, its
