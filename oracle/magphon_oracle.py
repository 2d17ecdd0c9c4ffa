"""CPU oracle for the coupled Maxwell-LLG time step.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may call it, and only as the
checker or the timed CPU baseline -- never as the thing measured or shipped.

This is a numpy restatement of the reference solver path of
``magphon`` (``/root/reference/pkg/src/magphon``), written to reproduce its
IEEE fp64 results bit for bit: every elementwise expression below performs
the same operations in the same order as the reference line it cites.

Parity pinned: ``tests/golden/make_golden.py`` runs the reference itself
(``magphon.sim.run``) on the golden configs and checks this module against it
with ``np.array_equal`` before writing ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` re-checks the oracle against those fixtures.

The config is duck-typed: any object with the attributes of the reference
``SimConfig`` (``grid``, ``materials``, ``source``, ``boundaries``,
``cfl_factor``, ``t_end``, ``probes``, ``bias_direction``, ``llg_params``)
works -- the reference's own objects and the product's mirror alike.
"""

from __future__ import annotations

import math
import time

import numpy as np

# constants.py:22-25
EPS0 = 8.8541878128e-12
MU0 = 4e-7 * math.pi
C0 = 299792458.0
GAMMA_E = -1.759e11

_FACE_ORDER = (("x0", 0, 0), ("x1", 0, 1), ("y0", 1, 0), ("y1", 1, 1),
               ("z0", 2, 0), ("z1", 2, 1))          # em.py:290-291
_TANGENTIAL = {0: (1, 2), 1: (0, 2), 2: (0, 1)}     # em.py:293 (E comp index)


class OracleStepFailure(RuntimeError):
    """Mirror of ``llg.StepFailure`` (llg.py:38-46) with the step attached."""

    def __init__(self, message, residual, iterations, step=None):
        super().__init__(message)
        self.residual = residual
        self.iterations = iterations
        self.step = step


# ---------------------------------------------------------------------------
# scalars
# ---------------------------------------------------------------------------

def cfl_dt(n, d, factor):
    """em.py:82-93 (same Python-float expression, incl. ``d**2``)."""
    inv2 = sum(1.0 / s**2 for s, c in zip(d, n) if c > 1)
    return factor / (C0 * math.sqrt(inv2))


def source_value(amplitude, f0, Tp, t):
    """em.py:96-101, evaluated left to right exactly as the reference."""
    env = math.exp(-((t - 3.0 * Tp) ** 2) / (2.0 * Tp**2))
    return amplitude * env * math.cos(2.0 * math.pi * f0 * t)


# ---------------------------------------------------------------------------
# state
# ---------------------------------------------------------------------------

class Lattice:
    """Field arrays in the reference allocation layout (grid.py:82-99)."""

    def __init__(self, n):
        self.n = tuple(n)
        fs = tuple(c + 1 if c > 1 else 1 for c in n)
        self.fs = fs
        self.E = [np.zeros(fs) for _ in range(3)]
        self.H = [np.zeros(fs) for _ in range(3)]
        self.M = np.zeros((3,) + self.n)

    def state(self):
        names = ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")
        return dict(zip(names, self.E + self.H)) | {"M": self.M}

    def load(self, st):
        for c, name in enumerate(("Ex", "Ey", "Ez")):
            self.E[c][...] = st[name]
        for c, name in enumerate(("Hx", "Hy", "Hz")):
            self.H[c][...] = st[name]
        self.M[...] = st["M"]

    def sample(self, comp, i, j, k):
        kind, c = comp[0], "xyz".index(comp[1])
        arr = {"E": self.E, "H": self.H}[kind][c] if kind != "M" else self.M[c]
        return float(arr[i, j, k])


def initial_magnetization(lat, Ms, Hbias):
    """grid.py:140-156: M = Ms * unit(Hbias) in magnetic cells, +x if 0."""
    mag = Ms > 0.0
    if mag.any():
        b = Hbias[:, mag]
        norm = np.sqrt((b * b).sum(axis=0))
        u = np.zeros_like(b)
        ok = norm > 0
        u[:, ok] = b[:, ok] / norm[ok]
        u[0, ~ok] = 1.0
        lat.M[:, mag] = Ms[mag] * u


def with_bias(Ms, Hbias, bias, direction):
    """sim.py:82-97: replace Hbias in Ms>0 cells by bias * unit(direction)."""
    Hb = Hbias.copy()
    mag = Ms > 0
    dv = np.asarray(direction, float)
    dv = dv / np.linalg.norm(dv)
    for c in range(3):
        Hb[c][mag] = bias * dv[c]
    return Hb


# ---------------------------------------------------------------------------
# stencils
# ---------------------------------------------------------------------------

def _fwd(a, axis, n, d):
    """em.py:108-114: (a[i+1]-a[i])/d over the first n entries of axis."""
    hi = [slice(None)] * 3
    lo = [slice(None)] * 3
    hi[axis] = slice(1, n + 1)
    lo[axis] = slice(0, n)
    return (a[tuple(hi)] - a[tuple(lo)]) / d


def curl_e(lat, d):
    """em.py:117-139 (accumulation into zero arrays kept for parity)."""
    nx, ny, nz = lat.n
    Ex, Ey, Ez = lat.E
    c = [np.zeros(lat.fs) for _ in range(3)]
    if ny > 1:
        c[0][:, :ny, :] += _fwd(Ez, 1, ny, d[1])
        c[2][:, :ny, :] -= _fwd(Ex, 1, ny, d[1])
    if nz > 1:
        c[0][:, :, :nz] -= _fwd(Ey, 2, nz, d[2])
        c[1][:, :, :nz] += _fwd(Ex, 2, nz, d[2])
    if nx > 1:
        c[1][:nx, :, :] -= _fwd(Ez, 0, nx, d[0])
        c[2][:nx, :, :] += _fwd(Ey, 0, nx, d[0])
    return c


def h_masks(lat, mag):
    """em.py:142-168: valid H ranges minus same-index magnetic cells."""
    nx, ny, nz = lat.n
    valid = ((slice(None), slice(0, ny), slice(0, nz)),
             (slice(0, nx), slice(None), slice(0, nz)),
             (slice(0, nx), slice(0, ny), slice(None)))
    out = []
    for v in valid:
        m = np.zeros(lat.fs, dtype=bool)
        m[v] = True
        m[:nx, :ny, :nz] &= ~mag
        out.append(m)
    return out


def _bwd_ghost(a, axis, n, d, pmc_lo, pmc_hi):
    """em.py:185-203: backward difference at n+1 nodes with PMC ghosts."""
    core = [slice(None)] * 3
    core[axis] = slice(0, n)
    body = a[tuple(core)]
    e = [slice(None)] * 3
    e[axis] = slice(0, 1)
    lo = -body[tuple(e)] if pmc_lo else np.zeros_like(body[tuple(e)])
    e[axis] = slice(n - 1, n)
    hi = -body[tuple(e)] if pmc_hi else np.zeros_like(body[tuple(e)])
    p = np.concatenate([lo, body, hi], axis=axis)
    s1 = [slice(None)] * 3
    s0 = [slice(None)] * 3
    s1[axis] = slice(1, n + 2)
    s0[axis] = slice(0, n + 1)
    return (p[tuple(s1)] - p[tuple(s0)]) / d


def curl_h(lat, d, faces):
    """em.py:206-232."""
    nx, ny, nz = lat.n
    Hx, Hy, Hz = lat.H
    pmc = {f: faces[f] == "PMC" for f in faces}
    c = [np.zeros(lat.fs) for _ in range(3)]
    if ny > 1:
        c[0] += _bwd_ghost(Hz, 1, ny, d[1], pmc["y0"], pmc["y1"])
        c[2] -= _bwd_ghost(Hx, 1, ny, d[1], pmc["y0"], pmc["y1"])
    if nz > 1:
        c[0] -= _bwd_ghost(Hy, 2, nz, d[2], pmc["z0"], pmc["z1"])
        c[1] += _bwd_ghost(Hx, 2, nz, d[2], pmc["z0"], pmc["z1"])
    if nx > 1:
        c[1] -= _bwd_ghost(Hz, 0, nx, d[0], pmc["x0"], pmc["x1"])
        c[2] += _bwd_ghost(Hy, 0, nx, d[0], pmc["x0"], pmc["x1"])
    return c


def _edge_pad(a, n):
    return np.pad(a, [(0, 1) if c > 1 else (0, 0) for c in n], mode="edge")


def e_coefficients(sigma, eps_r, n, dt):
    """em.py:239-254."""
    s = _edge_pad(sigma, n)
    eps = EPS0 * _edge_pad(eps_r, n)
    return 1.0 / (s / 2.0 + eps / dt), s / 2.0 - eps / dt


def _plane(a, axis, idx):
    sl = [slice(None)] * 3
    sl[axis] = idx
    return a[tuple(sl)]


def walls(lat, faces, d, dt, eps_r, prev):
    """em.py:324-359, faces strictly in the order x0,x1,y0,y1,z0,z1."""
    for face, axis, side in _FACE_ORDER:
        if lat.n[axis] <= 1:
            continue
        wall = 0 if side == 0 else lat.n[axis]
        cond = faces[face]
        if cond == "PEC":
            for c in _TANGENTIAL[axis]:
                _plane(lat.E[c], axis, wall)[...] = 0.0
        elif cond == "MUR1":
            inner = wall + (1 if side == 0 else -1)
            eps_w = EPS0 * _plane(_edge_pad(eps_r, lat.n), axis, wall)
            cl = 1.0 / np.sqrt(MU0 * eps_w)
            k = (cl * dt - d[axis]) / (cl * dt + d[axis])
            for c in _TANGENTIAL[axis]:
                pw, pi = prev[(face, c)]
                _plane(lat.E[c], axis, wall)[...] = (
                    pi + k * (_plane(lat.E[c], axis, inner) - pw))


def capture_mur(lat, faces):
    """em.py:306-321."""
    prev = {}
    for face, axis, side in _FACE_ORDER:
        if faces[face] != "MUR1":
            continue
        if lat.n[axis] <= 1:
            raise ValueError(f"MUR1 on collapsed axis face {face}")
        wall = 0 if side == 0 else lat.n[axis]
        inner = wall + (1 if side == 0 else -1)
        for c in _TANGENTIAL[axis]:
            prev[(face, c)] = (_plane(lat.E[c], axis, wall).copy(),
                               _plane(lat.E[c], axis, inner).copy())
    return prev


# ---------------------------------------------------------------------------
# LLG fixed point (llg.py:61-148)
# ---------------------------------------------------------------------------

def _cross(u, v):
    return np.stack((u[1] * v[2] - u[2] * v[1],
                     u[2] * v[0] - u[0] * v[2],
                     u[0] * v[1] - u[1] * v[0]))


def llg_iterates(Hn, Mn, Hbias, cE, dt, alpha, Ms, gamma, tol, max_iters,
                 per_cell=False):
    """llg.py:108-148.  Returns (H, M, iterations).

    With ``per_cell`` it also returns, per cell, the first iterate whose own
    residual is <= tol (0 if none) -- a diagnostic used by tests to make sure
    a golden exercises steps where magnetic cells disagree on convergence.
    """
    c = MU0 * np.abs(gamma) * dt / 2.0
    b = Mn - c * _cross(Mn, Hn + Hbias)
    coef = dt / MU0
    Hr, Mr = Hn, Mn
    prev = np.inf
    growth = 0
    first = np.zeros(Hn.shape[1:], dtype=int)
    for it in range(1, max_iters + 1):
        a = -(c * (Hr + Hbias) + (alpha / Ms) * Mn)
        adotb = (a * b).sum(axis=0)
        m = (b + adotb * a - _cross(a, b)) / (1.0 + (a * a).sum(axis=0))
        Mnew = m * (Ms / np.sqrt((m * m).sum(axis=0)))
        rc = np.abs(Mnew - Mr) / Ms
        res = float(np.max(rc))
        if per_cell:
            hit = (rc.max(axis=0) <= tol) & (first == 0)
            first[hit] = it
        Mr = Mnew
        Hr = Hn + (Mn - Mr) - coef * cE
        if res <= tol:
            return (Hr, Mr, it, first) if per_cell else (Hr, Mr, it)
        growth = growth + 1 if res > prev else 0
        if growth >= 3:
            raise OracleStepFailure(
                f"fixed-point iteration diverging (residual {res:.3e} after "
                f"{it} iterates)", res, it)
        prev = res
    raise OracleStepFailure(
        f"fixed-point iteration did not reach tol {tol:.1e} in {max_iters} "
        f"iterates (residual {prev:.3e})", prev, max_iters)


# ---------------------------------------------------------------------------
# run (sim.py:125-180)
# ---------------------------------------------------------------------------

def _faces(bnd):
    return {f: getattr(bnd, f) for f in ("x0", "x1", "y0", "y1", "z0", "z1")}


def run(config, bias=None, resume=None, n_steps=None, record_first=False, marks=None):
    """Restatement of ``sim.run``; returns a plain dict.

    ``n_steps`` (oracle-only) truncates the run for bounded CPU baselines;
    ``marks`` (a list) receives ``time.perf_counter()`` at the start of every
    step and once after the last, so a baseline can time the steps alone.
    """
    g = config.grid
    n = (g.nx, g.ny, g.nz)
    d = (g.dx, g.dy, g.dz)
    mats = config.materials
    sigma, eps_r = np.asarray(mats.sigma), np.asarray(mats.eps_r)
    Ms, alpha = np.asarray(mats.Ms), np.asarray(mats.alpha)
    gamma, Hbias = np.asarray(mats.gamma_e), np.asarray(mats.Hbias)
    if bias is not None:
        Hbias = with_bias(Ms, Hbias, bias, config.bias_direction)
    faces = _faces(config.boundaries)
    lat = Lattice(n)
    initial_magnetization(lat, Ms, Hbias)
    dt = cfl_dt(n, d, config.cfl_factor)
    total = int(np.ceil(config.t_end / dt))
    stop = total if n_steps is None else min(total, n_steps)
    mag = Ms > 0.0
    idx = np.nonzero(mag)
    any_mag = len(idx[0]) > 0
    if any_mag:
        mMs, malpha, mgamma = Ms[idx], alpha[idx], gamma[idx]
        mHb = np.stack([Hbias[c][idx] for c in range(3)])
    masks = h_masks(lat, mag)
    ca, cb = e_coefficients(sigma, eps_r, n, dt)
    coef = dt / MU0
    src = config.source
    probes = {(p[0], (p[1], p[2], p[3])): [] for p in config.probes}
    iters = []
    firsts = []
    start = 0
    if resume is not None:
        lat.load(resume["fields"])
        start = int(resume["step"])
        for key, vals in resume["probes"].items():
            probes[key] = list(vals)
        iters = list(resume["iterations"])
    tol, max_iters = config.llg_params.tol, config.llg_params.max_iters
    for step in range(start, stop):
        if marks is not None:
            marks.append(time.perf_counter())
        cE = curl_e(lat, d)
        for c in range(3):
            m = masks[c]
            lat.H[c][m] -= coef * cE[c][m]
        if any_mag:
            Hn = np.stack([lat.H[c][idx] for c in range(3)])
            Mn = lat.M[:, idx[0], idx[1], idx[2]]
            cEm = np.stack([cE[c][idx] for c in range(3)])
            try:
                out = llg_iterates(Hn, Mn, mHb, cEm, dt, malpha, mMs, mgamma,
                                   tol, max_iters, per_cell=record_first)
            except OracleStepFailure as exc:
                exc.step = step
                raise
            H1, M1, it = out[:3]
            if record_first:
                firsts.append(out[3])
            for c in range(3):
                lat.H[c][idx] = H1[c]
            lat.M[:, idx[0], idx[1], idx[2]] = M1
            iters.append(it)
        prev = capture_mur(lat, faces)
        cH = curl_h(lat, d, faces)
        for c in range(3):
            lat.E[c][...] = ca * (cH[c] - cb * lat.E[c])
        walls(lat, faces, d, dt, eps_r, prev)
        v = source_value(src.amplitude, src.f0, src.Tp, (step + 1) * dt)
        i, j, k = src.location
        for c, p in enumerate(src.polarization):
            if p != 0.0:
                lat.E[c][i, j, k] += p * v
        for (comp, loc), buf in probes.items():
            buf.append(lat.sample(comp, *loc))
    if marks is not None:
        marks.append(time.perf_counter())
    out = {
        "fields": lat.state(),
        "probes": {k: np.asarray(v) for k, v in probes.items()},
        "iterations": np.asarray(iters, dtype=int),
        "steps": stop,
        "dt": dt,
    }
    if record_first:
        out["first_converged"] = firsts
    return out


def total_energy(state, eps_r, Hbias, n, d):
    """em.py:366-383 on a state dict."""
    vol = d[0] * d[1] * d[2]
    eps = EPS0 * _edge_pad(np.asarray(eps_r), n)
    ue = 0.5 * float(sum(np.sum(eps * state[c] ** 2) for c in ("Ex", "Ey", "Ez")))
    uh = 0.5 * MU0 * float(sum(np.sum(state[c] ** 2) for c in ("Hx", "Hy", "Hz")))
    uz = -MU0 * float(np.sum(state["M"] * np.asarray(Hbias)))
    return (ue + uh + uz) * vol
