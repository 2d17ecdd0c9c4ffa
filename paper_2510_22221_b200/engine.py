"""Device engine: turns a run description into the C-ABI setup and drives it.

The engine owns one ``mpb_handle`` (device state of one run).  All per-cell
material data is compressed here to a uint8 material id per cell plus a
table of host-precomputed coefficients -- computed with the same numpy fp64
expressions the reference evaluates per entry, so the device multiplies
exactly the same doubles:

* ``ca, cb``   -- reference em.py:239-254
* ``mur_k``    -- reference em.py:352-357
* ``c_llg``    -- reference llg.py:125 (mu0*|gamma|*dt/2)
* ``alpha_ms`` -- reference llg.py:132 (alpha/Ms)
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .constants import CONSTANTS

E_H_NAMES = ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")


def _codes(arr: np.ndarray, limit: int = 64):
    """Small-alphabet encoding of an array with few distinct values.

    Returns (codes, values, first_index).  One vectorised pass per distinct
    value, so 1e8-cell maps with a handful of materials encode in seconds;
    falls back to np.unique beyond ``limit`` values.
    """
    flat = arr.reshape(-1)
    codes = np.full(flat.shape, -1, dtype=np.int32)
    values, firsts = [], []
    todo = np.ones(flat.shape, dtype=bool)
    start = 0
    while True:
        rest = np.flatnonzero(todo[start:start + (1 << 20)])
        if rest.size == 0:
            rest = np.flatnonzero(todo[start:])
            if rest.size == 0:
                break
        first = start + int(rest[0])
        v = flat[first]
        hit = np.isnan(flat) if v != v else (flat == v)
        codes[hit & todo] = len(values)
        values.append(v)
        firsts.append(first)
        todo &= ~hit
        start = first
        if len(values) > limit:
            u, idx, inv = np.unique(flat, return_index=True, return_inverse=True)
            return inv.astype(np.int32).reshape(arr.shape), list(u), list(idx)
    return codes.reshape(arr.shape), values, firsts


def magnetic_count(materials) -> int:
    if getattr(materials, "lazy", False):
        return materials.magnetic_count()
    return int(np.count_nonzero(np.asarray(materials.Ms) > 0.0))


def material_table(materials, dt: float, spacings):
    """Per-cell uint8 ids and the coefficient table for ``materials``."""
    if getattr(materials, "lazy", False):
        # painted map: ids straight from the boxes, one row per distinct cell
        ids, cells = materials.painted()
        if len(cells) > N.MAX_MATERIALS:
            raise ValueError(f"{len(cells)} distinct materials; the device table "
                             f"holds at most {N.MAX_MATERIALS}")
        col = lambda name: np.array([getattr(c, name) for c in cells], dtype=float)  # noqa: E731
        hb = np.array([c.Hbias for c in cells], dtype=float).T
        return ids, _table(col("sigma"), col("eps_r"), col("Ms"), col("alpha"),
                           col("gamma_e"), [hb[c] for c in range(3)],
                           col("Ms") > 0.0, dt, spacings)
    mag = np.asarray(materials.Ms) > 0.0
    fields = [np.asarray(materials.sigma), np.asarray(materials.eps_r)]
    mfields = [np.asarray(materials.Ms), np.asarray(materials.alpha),
               np.asarray(materials.gamma_e)] + [np.asarray(materials.Hbias[c])
                                                for c in range(3)]
    key = np.zeros(mag.shape, dtype=np.int64)
    radix = 1
    for a in fields:
        cd, vals, _ = _codes(a)
        key += cd.astype(np.int64) * radix
        radix *= len(vals)
    # magnetic parameters only matter in magnetic cells
    key = key * 2 + mag
    radix *= 2
    if mag.any():
        for a in mfields:
            sub = np.where(mag, a, 0.0)
            cd, vals, _ = _codes(sub)
            key += cd.astype(np.int64) * radix
            radix *= max(1, len(vals))
    inv, ukeys, first = _codes(key, limit=N.MAX_MATERIALS)
    nmat = len(ukeys)
    if nmat > N.MAX_MATERIALS:
        raise ValueError(f"{nmat} distinct materials; the device table "
                         f"holds at most {N.MAX_MATERIALS}")
    first = np.asarray(first)
    ids = inv.astype(np.uint8).reshape(mag.shape)
    pick = lambda a: np.asarray(a).reshape(-1)[first]     # noqa: E731
    sigma, eps_r = pick(fields[0]), pick(fields[1])
    Ms, alpha, gamma = pick(mfields[0]), pick(mfields[1]), pick(mfields[2])
    hb = [pick(materials.Hbias[c]) for c in range(3)]
    ismag = pick(mag)
    return ids, _table(sigma, eps_r, Ms, alpha, gamma, hb, ismag, dt, spacings)


def _table(sigma, eps_r, Ms, alpha, gamma, hb, ismag, dt, spacings):
    """Coefficient rows from per-material parameter vectors."""
    nmat = len(sigma)
    # --- coefficients, reference expressions verbatim in meaning/order ---
    eps = CONSTANTS.eps0 * eps_r
    ca = 1.0 / (sigma / 2.0 + eps / dt)
    cb = sigma / 2.0 - eps / dt
    cl = 1.0 / np.sqrt(CONSTANTS.mu0 * eps)
    with np.errstate(divide="ignore", invalid="ignore"):
        c_llg = CONSTANTS.mu0 * np.abs(gamma) * dt / 2.0
        a_ms = np.where(ismag, alpha / np.where(ismag, Ms, 1.0), 0.0)
    table = (N.Material * nmat)()
    for q in range(nmat):
        m = table[q]
        m.ca, m.cb = ca[q], cb[q]
        for a in range(3):
            m.mur_k[a] = (cl[q] * dt - spacings[a]) / (cl[q] * dt + spacings[a])
        m.Ms = Ms[q]
        m.alpha_ms = a_ms[q]
        m.c_llg = c_llg[q]
        for c in range(3):
            m.hbias[c] = hb[c][q]
        m.magnetic = int(bool(ismag[q]))
        m.eps = eps[q]
    return table


class DeviceRun:
    """One run's device state behind the C ABI (one handle)."""

    def __init__(self, grid, materials, boundaries, source_loc, source_pol,
                 probes, llg_params, dt: float, device: int = 0,
                 kernel_variant: int = 0, graph_steps: int = 0, slab=None,
                 storage: str = "f64"):
        """``slab``: None (whole grid on one GPU) or a ``parallel.Slab``
        (multi-rank x-slab); ``materials`` then covers the slab's cell
        planes incl. ghosts (``Slab.cell_range``), ``grid`` is global.
        ``storage``: "f64" (reference precision, bit-exact) or "f32" (E/H in
        fp32 on the device, M and the LLG in fp64; within tolerance)."""
        if storage not in N.STORAGE_CODES:
            raise ValueError(f"storage must be one of {sorted(N.STORAGE_CODES)}")
        self.storage = storage
        self.lib = N.load_library()
        self.grid = grid
        self.n = grid.cell_shape
        self.fs = grid.field_shape
        self.slab = slab
        if slab is not None:
            f0, f1 = slab.field_range
            c0, c1 = slab.cell_range
            self.fs = (f1 - f0,) + tuple(self.fs[1:])
            self.n = (c1 - c0,) + tuple(self.n[1:])
        self.probes = list(probes)
        ids, table = material_table(materials, dt, grid.spacings)
        self._keep = [ids, table]
        su = N.Setup()
        su.n[:] = list(grid.cell_shape)          # global grid; slabs carry ranges
        su.d[:] = list(grid.spacings)
        su.dt = dt
        su.coef_h = dt / CONSTANTS.mu0
        su.faces[:] = [N.FACE_CODES[getattr(boundaries, f)]
                       for f in ("x0", "x1", "y0", "y1", "z0", "z1")]
        su.n_materials = len(table)
        su.materials = C.cast(table, C.POINTER(N.Material))
        idc = np.ascontiguousarray(ids)
        self._keep.append(idc)
        su.cell_material = idc.ctypes.data_as(C.POINTER(C.c_uint8))
        su.src_loc[:] = list(source_loc)
        su.src_pol[:] = [float(p) for p in source_pol]
        comp = np.array([N.COMP_CODES[p[0]] for p in self.probes] or [0],
                        dtype=np.int32)
        loc = np.array([list(p[1]) for p in self.probes] or [[0, 0, 0]],
                       dtype=np.int32).reshape(-1)
        self._keep += [comp, loc]
        su.n_probes = len(self.probes)
        su.probe_comp = comp.ctypes.data_as(C.POINTER(C.c_int32))
        su.probe_loc = loc.ctypes.data_as(C.POINTER(C.c_int32))
        su.llg_tol = llg_params.tol
        su.llg_max_iters = llg_params.max_iters
        su.device = device
        su.kernel_variant = kernel_variant
        su.graph_steps = graph_steps
        su.storage = N.STORAGE_CODES[storage]
        n_magnetic = magnetic_count(materials)
        if slab is None:
            su.nranks, su.rank, su.x_lo, su.x_hi = 1, 0, 0, grid.nx
            su.any_magnetic = int(n_magnetic > 0)
        else:
            su.nranks, su.rank = slab.nranks, slab.rank
            su.x_lo, su.x_hi = slab.x_lo, slab.x_hi
            su.any_magnetic = int(slab.any_magnetic)
            su.nccl_id[:] = list(slab.nccl_id)
        h = C.c_void_p()
        N.check(self.lib.mpb_create(C.byref(su), C.byref(h)))
        self.h = h
        self.n_magnetic = n_magnetic

    # -- state ---------------------------------------------------------------
    def load_state(self, fields: dict | None, M: np.ndarray) -> None:
        """``fields`` None: E and H start at zero (no host arrays)."""
        if fields is None:
            arrs = [None] * 6
        else:
            arrs = [np.ascontiguousarray(fields[n], dtype=np.float64) for n in E_H_NAMES]
            for a in arrs:
                if a.shape != self.fs:
                    raise ValueError("snapshot shape mismatch")
        m = np.ascontiguousarray(M, dtype=np.float64)
        if m.shape != (3,) + tuple(self.n):
            raise ValueError("snapshot shape mismatch for M")
        ptrs = (C.POINTER(C.c_double) * 6)(
            *[a.ctypes.data_as(C.POINTER(C.c_double)) if a is not None else None
              for a in arrs])
        N.check(self.lib.mpb_load_state(self.h, ptrs,
                                        m.ctypes.data_as(C.POINTER(C.c_double))))

    def save_state(self) -> dict:
        out = {n: np.empty(self.fs) for n in E_H_NAMES}
        M = np.empty((3,) + tuple(self.n))
        ptrs = (C.POINTER(C.c_double) * 6)(
            *[out[n].ctypes.data_as(C.POINTER(C.c_double)) for n in E_H_NAMES])
        N.check(self.lib.mpb_save_state(self.h, ptrs,
                                        M.ctypes.data_as(C.POINTER(C.c_double))))
        out["M"] = M
        return out

    # -- stepping ------------------------------------------------------------
    def run(self, n0: int, src_vals: np.ndarray, probes: np.ndarray | None = None,
            iters: np.ndarray | None = None):
        """Advance len(src_vals) steps.  Returns (probes[steps, P], iters,
        failure) with failure None or (step, residual, iterations, kind).
        ``probes`` / ``iters`` may be caller-provided (e.g. pinned) host
        arrays of shape (steps, max(1, P)) float64 / (steps,) int32."""
        src = np.ascontiguousarray(src_vals, dtype=np.float64)
        steps = src.size
        if probes is None:
            probes = np.zeros((steps, max(1, len(self.probes))))
        if iters is None:
            iters = np.zeros(steps, dtype=np.int32)
        if (probes.shape != (steps, max(1, len(self.probes))) or probes.dtype != np.float64
                or not probes.flags.c_contiguous or iters.shape != (steps,)
                or iters.dtype != np.int32):
            raise ValueError("probe / iteration buffers do not match the run")
        fail = N.Failure()
        code = self.lib.mpb_run(self.h, n0, steps,
                                src.ctypes.data_as(C.POINTER(C.c_double)),
                                probes.ctypes.data_as(C.POINTER(C.c_double)),
                                iters.ctypes.data_as(C.POINTER(C.c_int32)),
                                C.byref(fail))
        if code == N.ESTEP:
            return probes[:, :len(self.probes)], iters, (
                int(fail.step), float(fail.residual), int(fail.iterations),
                int(fail.kind))
        N.check(code)
        return probes[:, :len(self.probes)], iters, None

    def run_device(self, n0: int, nsteps: int, d_src: int, d_probe: int,
                   d_iters: int, stream: int = 0) -> None:
        N.check(self.lib.mpb_run_device(self.h, n0, nsteps, C.c_void_p(d_src),
                                        C.c_void_p(d_probe), C.c_void_p(d_iters),
                                        C.c_void_p(stream)))

    def check_failure(self):
        fail = N.Failure()
        code = self.lib.mpb_check_failure(self.h, C.byref(fail))
        if code == N.ESTEP:
            return (int(fail.step), float(fail.residual), int(fail.iterations),
                    int(fail.kind))
        N.check(code)
        return None

    def set_kernel_timing(self, on: bool) -> None:
        N.check(self.lib.mpb_set_kernel_timing(self.h, int(on)))

    def kernel_time(self):
        ms = C.c_double()
        cnt = C.c_int64()
        name = C.c_char_p()
        N.check(self.lib.mpb_kernel_time(self.h, C.byref(ms), C.byref(cnt),
                                         C.byref(name)))
        return ms.value, cnt.value, name.value.decode()

    def total_energy(self) -> float:
        """em.total_energy of the current device state (this rank's planes)."""
        out = C.c_double()
        N.check(self.lib.mpb_total_energy(self.h, C.byref(out)))
        return out.value

    def sweep_form(self) -> dict:
        """Tile form of the fused sweep (V, NT, T, x-chunks)."""
        out = (C.c_int32 * 4)()
        N.check(self.lib.mpb_sweep_form(self.h, out))
        return {"V": out[0], "NT": out[1], "T": out[2], "chunks": out[3]}

    def comm_info(self) -> dict:
        """Ranks as the NCCL communicator reports them + the NCCL version."""
        n, r, v = C.c_int32(), C.c_int32(), C.c_int32()
        N.check(self.lib.mpb_comm_info(self.h, C.byref(n), C.byref(r), C.byref(v)))
        return {"nranks": n.value, "rank": r.value, "nccl_version": v.value}

    def launch_count(self) -> int:
        return int(self.lib.mpb_launch_count(self.h))

    def device_bytes(self) -> int:
        return int(self.lib.mpb_device_bytes(self.h))

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.mpb_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
