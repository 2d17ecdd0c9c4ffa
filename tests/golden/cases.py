"""Golden parity cases, described as plain data.

The same description is built into a config by the reference package (only
in ``make_golden.py``, in the build container where ``/root/reference``
exists) and by this repo's own host mirror (in the tests, anywhere).  Both
expose the reference API names (GridSpec, MaterialMap, MaterialCell,
SourceSpec, BoundarySpec, LlgIterationParams, SimConfig), so one builder
serves both.
"""

from __future__ import annotations

OE = 1000.0 / (4.0 * 3.141592653589793)   # only for readable case tables

CASES = {
    # 3D, every boundary type, a conductor layer, a dielectric, a magnet
    # whose steps need r* = 1 and 2, strong source (SURVEY Appendix A grid).
    "mixed3d": dict(
        grid=(12, 10, 14, 10e-6, 8e-6, 6e-6),
        background=(0.0, 2.0),
        boxes=[
            dict(box=(0, 12, 0, 10, 0, 3), eps_r=11.4),
            dict(box=(0, 12, 0, 10, 3, 4), sigma=1e6),
            dict(box=(5, 8, 4, 7, 6, 9), eps_r=15.0, Ms=1.3926e5,
                 alpha=1e-3, bias=1000.0 * OE, bias_direction=(0, 0, 1)),
        ],
        source=dict(f0=50e9, Tp=1e-12, amplitude=1e7, location=(4, 5, 7),
                    polarization=(0.0, 1.0, 0.0)),
        boundaries=dict(x0="PMC", x1="MUR1", y0="PEC", y1="PMC", z0="MUR1",
                        z1="PEC"),
        cfl=0.9, steps=120,
        probes=[("Ey", 4, 5, 8), ("Hx", 6, 5, 7), ("Mx", 6, 5, 7),
                ("Mz", 6, 5, 7), ("Ez", 12, 3, 3)],
    ),
    # all-MUR1 box, source next to a corner: wall order is observable here
    "allmur3d": dict(
        grid=(10, 9, 11, 5e-6, 5e-6, 5e-6),
        background=(0.0, 1.0),
        boxes=[dict(box=(4, 7, 3, 6, 4, 8), eps_r=15.0, Ms=9.7e5, alpha=0.01,
                    bias=2000.0 * OE, bias_direction=(1, 1, 0))],
        source=dict(f0=80e9, Tp=0.5e-12, amplitude=1e6, location=(1, 1, 1),
                    polarization=(0.0, 0.0, 1.0)),
        boundaries=dict(x0="MUR1", x1="MUR1", y0="MUR1", y1="MUR1",
                        z0="MUR1", z1="MUR1"),
        cfl=0.95, steps=200,
        probes=[("Ez", 1, 1, 2), ("My", 5, 4, 5), ("Hy", 0, 0, 0),
                # M outside the magnet (a constant) and an H padding entry
                ("Mz", 0, 0, 0), ("Hz", 10, 9, 0), ("Ex", 9, 9, 11)],
    ),
    # C1 in miniature: PEC box, YIG block, strong drive (mixed per-cell r_c)
    "pec_block": dict(
        grid=(16, 16, 16, 10e-6, 10e-6, 10e-6),
        background=(0.0, 1.0),
        boxes=[dict(box=(6, 10, 6, 10, 6, 10), eps_r=15.0, Ms=1.3926e5,
                    alpha=1e-3, bias=1000.0 * OE, bias_direction=(0, 0, 1))],
        source=dict(f0=50e9, Tp=1e-12, amplitude=1e8, location=(4, 8, 8),
                    polarization=(0.0, 1.0, 0.0)),
        boundaries=dict(x0="PEC", x1="PEC", y0="PEC", y1="PEC", z0="PEC",
                        z1="PEC"),
        cfl=0.9, steps=150,
        probes=[("Ey", 5, 8, 8), ("Hx", 8, 8, 8), ("Mx", 8, 8, 8),
                ("My", 8, 8, 8), ("Mz", 8, 8, 8)],
    ),
    # pec_block with a tolerance at which the global residual is
    # NON-MONOTONE in some steps (6 and 14): a cell whose own residual fell
    # below tol at iterate 1 is back above it at iterate 2, so the reference
    # keeps iterating past the last local stop (llg.py:131-148) -- the case
    # the multi-rank continuation (recover_suspended) exists for
    "nonmono3d": dict(
        grid=(16, 16, 16, 10e-6, 10e-6, 10e-6),
        background=(0.0, 1.0),
        boxes=[dict(box=(6, 10, 6, 10, 6, 10), eps_r=15.0, Ms=1.3926e5,
                    alpha=1e-3, bias=1000.0 * OE, bias_direction=(0, 0, 1))],
        source=dict(f0=50e9, Tp=1e-12, amplitude=1e8, location=(4, 8, 8),
                    polarization=(0.0, 1.0, 0.0)),
        boundaries=dict(x0="PEC", x1="PEC", y0="PEC", y1="PEC", z0="PEC",
                        z1="PEC"),
        cfl=0.9, steps=150, llg=(5.5e-8, 50),
        probes=[("Ey", 5, 8, 8), ("Hx", 8, 8, 8), ("Mx", 8, 8, 8),
                ("My", 8, 8, 8), ("Mz", 8, 8, 8)],
    ),
    # 2D (collapsed z): PMC/MUR/PEC in-plane faces
    "plane2d": dict(
        grid=(14, 12, 1, 4e-6, 6e-6, 3e-6),
        background=(1e-2, 3.0),
        boxes=[dict(box=(5, 9, 4, 8, 0, 1), eps_r=15.0, Ms=9.7e5, alpha=3e-3,
                    bias=1800.0 * OE, bias_direction=(1, 0, 0))],
        source=dict(f0=30e9, Tp=2e-12, amplitude=1e6, location=(3, 3, 0),
                    polarization=(0.6, 0.8, 0.0)),
        boundaries=dict(x0="MUR1", x1="PEC", y0="PMC", y1="MUR1"),
        cfl=0.9, steps=150,
        probes=[("Ex", 6, 6, 0), ("Hz", 6, 6, 0), ("Mz", 6, 6, 0)],
    ),
    # 1D along x (collapsed y, z)
    "xline1d": dict(
        grid=(60, 1, 1, 2e-6, 2e-6, 2e-6),
        background=(1e-4, 8.0),
        boxes=[dict(box=(30, 31, 0, 1, 0, 1), sigma=1e-3, eps_r=1.0, Ms=9.7e5,
                    alpha=0.003, bias=1855.3 * OE, bias_direction=(0, 1, 0))],
        source=dict(f0=14.3e9, Tp=1e-12, amplitude=1e6, location=(5, 0, 0),
                    polarization=(0.0, 0.0, 1.0)),
        boundaries=dict(x0="PMC", x1="MUR1"),
        cfl=1.0, steps=300,
        probes=[("Ez", 10, 0, 0), ("Mx", 30, 0, 0)],
    ),
    # the shipped 1D cavity (pkg/configs/cavity1d.cfg values), a prefix
    "cavity1d": dict(
        grid=(1, 1, 1835, 2e-6, 2e-6, 2e-6),
        background=(1.2520467594271872e-4, 8.168870103908924),
        boxes=[dict(box=(0, 1, 0, 1, 917, 918), sigma=1e-3, eps_r=1.0,
                    Ms=9.7e5, alpha=0.003, bias=1855.3 * OE,
                    bias_direction=(1, 0, 0))],
        source=dict(f0=14.3e9, Tp=50e-12, amplitude=1e3, location=(0, 0, 50),
                    polarization=(1.0, 0.0, 0.0)),
        boundaries=dict(z0="PMC", z1="PMC"),
        cfl=0.9, steps=2000,
        probes=[("Ex", 0, 0, 300), ("Mz", 0, 0, 917)],
    ),
    # the reference's own run-level fixture shape (test_simulation.py:10-25)
    # with a strong drive so the magnet is reached and r* = 2 occurs
    "small1d_strong": dict(
        grid=(1, 1, 120, 2e-6, 2e-6, 2e-6),
        background=(1e-4, 8.0),
        boxes=[dict(box=(0, 1, 0, 1, 60, 61), sigma=1e-3, eps_r=1.0, Ms=9.7e5,
                    alpha=0.003, bias=1855.3 * OE, bias_direction=(1, 0, 0))],
        source=dict(f0=14.3e9, Tp=1e-12, amplitude=1e7, location=(0, 0, 10),
                    polarization=(1.0, 0.0, 0.0)),
        boundaries=dict(z0="PMC", z1="PMC"),
        cfl=0.9, steps=400,
        probes=[("Ex", 0, 0, 20), ("Mz", 0, 0, 60), ("Hy", 0, 0, 60)],
    ),
    # fault injection: tolerance no iterate can meet in one step
    "fail_tol": dict(
        expect_failure=True,
        grid=(1, 1, 120, 2e-6, 2e-6, 2e-6),
        background=(1e-4, 8.0),
        boxes=[dict(box=(0, 1, 0, 1, 60, 61), sigma=1e-3, eps_r=1.0, Ms=9.7e5,
                    alpha=0.003, bias=1855.3 * OE, bias_direction=(1, 0, 0))],
        source=dict(f0=14.3e9, Tp=1e-12, amplitude=1e3, location=(0, 0, 10),
                    polarization=(1.0, 0.0, 0.0)),
        boundaries=dict(z0="PMC", z1="PMC"),
        cfl=0.9, steps=400, llg=(1e-16, 1),
        probes=[("Ex", 0, 0, 20)],
    ),
    # magnet spanning the full z extent (touches both z walls, MUR1) under a
    # strong drive: deferred E recompute through z-wall rows
    "zwall_magnet": dict(
        grid=(8, 7, 6, 6e-6, 7e-6, 5e-6),
        background=(0.0, 2.0),
        boxes=[dict(box=(3, 6, 2, 5, 0, 6), eps_r=15.0, Ms=1.3926e5, alpha=2e-3,
                    bias=900.0 * OE, bias_direction=(1, 0, 1))],
        source=dict(f0=60e9, Tp=0.8e-12, amplitude=1e8, location=(2, 3, 1),
                    polarization=(0.6, 0.0, 0.8)),
        boundaries=dict(x0="PEC", x1="MUR1", y0="PMC", y1="MUR1", z0="MUR1",
                        z1="MUR1"),
        cfl=0.9, steps=150,
        probes=[("Ex", 4, 3, 0), ("Ey", 4, 3, 6), ("Mz", 4, 3, 0), ("Hx", 4, 3, 5)],
    ),
    # thinnest grid: ny = nz = 2, all MUR1 (z-wall inner rows coincide)
    "thin": dict(
        grid=(6, 2, 2, 4e-6, 4e-6, 4e-6),
        background=(0.0, 1.0),
        boxes=[dict(box=(2, 4, 0, 2, 0, 2), eps_r=15.0, Ms=9.7e5, alpha=5e-3,
                    bias=1500.0 * OE, bias_direction=(0, 0, 1))],
        source=dict(f0=80e9, Tp=0.5e-12, amplitude=1e7, location=(1, 1, 1),
                    polarization=(1.0, 0.0, 0.0)),
        boundaries=dict(x0="MUR1", x1="MUR1", y0="MUR1", y1="MUR1", z0="MUR1",
                        z1="MUR1"),
        cfl=0.9, steps=200,
        probes=[("Ex", 1, 1, 1), ("Ey", 3, 0, 0), ("My", 2, 1, 1)],
    ),
    # 1D along y (collapsed x, z): the sweep with one-entry rows (Fz = 1)
    "yline1d": dict(
        grid=(1, 50, 1, 3e-6, 3e-6, 3e-6),
        background=(2e-4, 6.0),
        boxes=[dict(box=(0, 1, 25, 26, 0, 1), sigma=1e-3, eps_r=1.0, Ms=9.7e5,
                    alpha=0.003, bias=1700.0 * OE, bias_direction=(1, 0, 1))],
        source=dict(f0=14.3e9, Tp=1e-12, amplitude=3e6, location=(0, 6, 0),
                    polarization=(0.0, 0.0, 1.0)),
        boundaries=dict(y0="MUR1", y1="PMC"),
        cfl=0.95, steps=300,
        probes=[("Ez", 0, 12, 0), ("Ex", 0, 30, 0), ("Mx", 0, 25, 0), ("Hy", 0, 24, 0)],
    ),
    # 2D in x-z (collapsed y): one-entry row halo, z walls with MUR1
    "plane_xz": dict(
        grid=(10, 1, 12, 5e-6, 5e-6, 4e-6),
        background=(0.0, 2.5),
        boxes=[dict(box=(4, 7, 0, 1, 5, 8), eps_r=15.0, Ms=1.3926e5, alpha=2e-3,
                    bias=1200.0 * OE, bias_direction=(0, 1, 0))],
        source=dict(f0=50e9, Tp=1e-12, amplitude=1e7, location=(2, 0, 3),
                    polarization=(0.0, 1.0, 0.0)),
        boundaries=dict(x0="PMC", x1="MUR1", z0="MUR1", z1="PEC"),
        cfl=0.9, steps=150,
        probes=[("Ey", 5, 0, 6), ("Hx", 5, 0, 6), ("My", 5, 0, 6), ("Ex", 0, 0, 0)],
    ),
    # the benchmark geometry in miniature: CPW strip + grounds as 1e11 S/m
    # boxes on a Si substrate, YIG film on the strip, all-MUR1 walls
    "cpw_small": dict(
        grid=(20, 24, 16, 10e-6, 10e-6, 2e-6),
        background=(0.0, 1.0),
        boxes=[dict(box=(0, 20, 0, 24, 0, 6), eps_r=11.4),
               dict(box=(0, 20, 0, 9, 6, 7), sigma=1e11),
               dict(box=(0, 20, 15, 24, 6, 7), sigma=1e11),
               dict(box=(0, 20, 11, 13, 6, 7), sigma=1e11),
               dict(box=(5, 15, 11, 13, 7, 9), eps_r=15.0, Ms=1.3926e5, alpha=1e-3,
                    bias=1000.0 * OE, bias_direction=(1, 0, 0))],
        source=dict(f0=60e9, Tp=0.5e-12, amplitude=1e8, location=(3, 10, 6),
                    polarization=(0.0, 1.0, 0.0)),
        boundaries=dict(x0="MUR1", x1="MUR1", y0="MUR1", y1="MUR1", z0="MUR1",
                        z1="MUR1"),
        cfl=0.9, steps=150,
        probes=[("Ey", 3, 10, 6), ("Ex", 10, 12, 7), ("Mz", 10, 12, 8), ("Hy", 10, 12, 8)],
    ),
    # two magnets of different materials and bias directions, conductor
    # between them, mixed walls, very strong drive
    "two_magnets": dict(
        grid=(14, 12, 10, 6e-6, 5e-6, 4e-6),
        background=(1e-3, 2.0),
        boxes=[dict(box=(2, 5, 3, 7, 2, 6), eps_r=15.0, Ms=9.7e5, alpha=3e-3,
                    bias=1900.0 * OE, bias_direction=(0, 1, 0)),
               dict(box=(6, 8, 0, 12, 0, 10), sigma=5e5),
               dict(box=(9, 13, 4, 9, 3, 8), eps_r=13.0, Ms=1.3926e5, alpha=1e-2,
                    bias=700.0 * OE, bias_direction=(1, 0, 1))],
        source=dict(f0=70e9, Tp=0.6e-12, amplitude=3e8, location=(5, 6, 5),
                    polarization=(0.0, 0.6, 0.8)),
        boundaries=dict(x0="PMC", x1="MUR1", y0="PEC", y1="MUR1", z0="PMC",
                        z1="MUR1"),
        cfl=0.9, steps=120,
        probes=[("Ez", 5, 6, 5), ("Mx", 3, 5, 4), ("My", 11, 6, 5), ("Hz", 10, 6, 5)],
    ),
    # StepFailure in 3D: many magnetic cells, a budget of 2 iterates and a
    # tolerance no step can meet (the failure comes from the global rule)
    "fail3d": dict(
        expect_failure=True,
        grid=(9, 8, 7, 6e-6, 6e-6, 5e-6),
        background=(0.0, 1.5),
        boxes=[dict(box=(2, 7, 2, 6, 2, 5), eps_r=15.0, Ms=1.3926e5, alpha=1e-3,
                    bias=1000.0 * OE, bias_direction=(0, 0, 1))],
        source=dict(f0=60e9, Tp=0.5e-12, amplitude=1e8, location=(1, 4, 3),
                    polarization=(0.0, 1.0, 0.0)),
        boundaries=dict(x0="MUR1", x1="PEC", y0="PMC", y1="MUR1", z0="PEC", z1="MUR1"),
        cfl=0.9, steps=100, llg=(1e-13, 2),
        probes=[("Ey", 1, 4, 3), ("Mx", 4, 4, 3)],
    ),
    # bias override through run(bias=...) along a tilted sweep direction
    "bias3d": dict(
        grid=(8, 9, 10, 6e-6, 6e-6, 6e-6),
        background=(0.0, 1.0),
        boxes=[dict(box=(2, 6, 3, 6, 3, 7), eps_r=15.0, Ms=1.3926e5,
                    alpha=2e-3, bias=500.0 * OE, bias_direction=(1, 0, 0))],
        source=dict(f0=40e9, Tp=1e-12, amplitude=3e7, location=(1, 4, 5),
                    polarization=(0.0, 0.0, 1.0)),
        boundaries=dict(x0="PEC", x1="MUR1", y0="PMC", y1="PEC", z0="MUR1",
                        z1="PMC"),
        cfl=0.9, steps=100, bias=2400.0 * OE, sweep_dir=(0.0, 1.0, 1.0),
        probes=[("Ez", 1, 4, 5), ("My", 3, 4, 4), ("Mz", 3, 4, 4)],
    ),
}


def build(case, ns):
    """Build a SimConfig for ``case`` with the API namespace ``ns``.

    ``ns`` maps GridSpec, MaterialCell, MaterialMap, SourceSpec, BoundarySpec,
    LlgIterationParams, SimConfig to classes (reference or mirror).
    """
    nx, ny, nz, dx, dy, dz = case["grid"]
    grid = ns["GridSpec"](nx, ny, nz, dx, dy, dz)
    sig, eps = case["background"]
    mm = ns["MaterialMap"](grid.cell_shape,
                           ns["MaterialCell"](sigma=sig, eps_r=eps))
    for b in case["boxes"]:
        dvec = b.get("bias_direction", (1, 0, 0))
        nrm = sum(x * x for x in dvec) ** 0.5
        hb = tuple(b.get("bias", 0.0) * x / nrm for x in dvec)
        cell = ns["MaterialCell"](sigma=b.get("sigma", 0.0),
                                  eps_r=b.get("eps_r", 1.0),
                                  Ms=b.get("Ms", 0.0),
                                  alpha=b.get("alpha", 0.0), Hbias=hb)
        mm.fill_box(cell, *b["box"])
    mm.freeze()
    src = ns["SourceSpec"](**case["source"])
    bnd = ns["BoundarySpec"](**case["boundaries"])
    tol, mx = case.get("llg", (1e-6, 50))
    cfg0 = ns["SimConfig"](
        grid=grid, materials=mm, source=src, boundaries=bnd,
        cfl_factor=case["cfl"], t_end=1.0,
        probes=tuple(tuple(p) for p in case["probes"]),
        bias_direction=tuple(case.get("sweep_dir", (1.0, 0.0, 0.0))),
        llg_params=ns["LlgIterationParams"](tol=tol, max_iters=mx))
    # t_end chosen so that ceil(t_end/dt) == steps exactly
    dt = cfg0.dt
    t_end = (case["steps"] - 0.5) * dt
    fields = {f: getattr(cfg0, f) for f in (
        "grid", "materials", "source", "boundaries", "cfl_factor", "probes",
        "bias_direction", "llg_params")}
    return ns["SimConfig"](t_end=t_end, **fields)


def reference_namespace():
    from magphon import em, llg, sim
    from magphon.grid import GridSpec
    from magphon.materials import MaterialCell, MaterialMap
    return dict(GridSpec=GridSpec, MaterialCell=MaterialCell,
                MaterialMap=MaterialMap, SourceSpec=em.SourceSpec,
                BoundarySpec=em.BoundarySpec,
                LlgIterationParams=llg.LlgIterationParams,
                SimConfig=sim.SimConfig)


def mirror_namespace():
    from paper_2510_22221_b200 import em, llg, sim
    from paper_2510_22221_b200.grid import GridSpec
    from paper_2510_22221_b200.materials import MaterialCell, MaterialMap
    return dict(GridSpec=GridSpec, MaterialCell=MaterialCell,
                MaterialMap=MaterialMap, SourceSpec=em.SourceSpec,
                BoundarySpec=em.BoundarySpec,
                LlgIterationParams=llg.LlgIterationParams,
                SimConfig=sim.SimConfig)
