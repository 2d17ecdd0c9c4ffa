"""Multi-rank NCCL code path on one GPU, with tests/nccl_emul/libnccl_emul.so
LD_PRELOADed in place of NCCL (tests/test_nccl_emul_gpu.py): each rank is a
handle created with a real NCCL id and driven by its own host thread through
mpb_run -- the library's exchange(), ncclCommSplit exchange communicator,
LLG all-reduces and suspended-step continuation all run, against the
reference goldens bit for bit.

    LD_PRELOAD=.../libnccl_emul.so python tests/nccl_emul_worker.py NRANKS case...
"""

import os
import sys
import threading
from dataclasses import replace

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2510_22221_b200 import _native as N  # noqa: E402
from paper_2510_22221_b200 import parallel  # noqa: E402
from paper_2510_22221_b200.grid import initial_magnetization  # noqa: E402
from paper_2510_22221_b200.sim import _materials_with_bias, source_values  # noqa: E402
from tests.golden.cases import CASES, build, mirror_namespace  # noqa: E402
from tests.golden_io import load  # noqa: E402


def nccl_id() -> bytes:
    import ctypes as C
    raw = (C.c_uint8 * 128)()
    N.check(N.load_library().mpb_nccl_unique_id(raw))
    return bytes(raw)


def run_case(name: str, nranks: int) -> str:
    case = CASES[name]
    g = load(name)
    config = build(case, mirror_namespace())
    bias = case.get("bias")
    materials = config.materials if bias is None else _materials_with_bias(
        config.materials, bias, config.bias_direction)
    keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in config.probes))
    any_mag = bool(np.count_nonzero(np.asarray(materials.Ms) > 0))
    nid = nccl_id()
    slabs = [replace(s, nccl_id=nid) for s in parallel.make_slabs(config.grid.nx, nranks, any_mag)]
    runs = parallel.slab_device_runs(config, materials, keys, slabs)
    names = ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")
    try:
        version = runs[0].comm_info()["nccl_version"]
        assert version == 99999, f"NCCL is not the emulation (version {version})"
        zeros = np.zeros(config.grid.field_shape)
        state = dict({n: zeros for n in names}, M=initial_magnetization(materials))
        for r, sl in zip(runs, slabs):
            r.load_state({n: parallel.local_fields(sl, state[n]) for n in names},
                         parallel.local_cells(sl, state["M"], axis=1))
        src = source_values(config.source, config.dt, 0, config.n_steps)
        out = [None] * nranks
        errs = []

        def go(q):
            try:
                out[q] = runs[q].run(0, src)
            except Exception as exc:   # reported by the main thread
                errs.append(exc)

        threads = [threading.Thread(target=go, args=(q,)) for q in range(nranks)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errs:
            raise errs[0]
        fails = [o[2] for o in out if o[2] is not None]
        if case.get("expect_failure"):
            assert fails, f"{name}: expected a StepFailure"
            step, res, it, kind = fails[0]
            assert step == int(g["fail_step"]) and it == int(g["fail_iterations"]), fails[0]
            assert res == float(g["fail_residual"]), fails[0]
            return f"OK {name} x{nranks} failure at step {step}"
        assert not fails, f"{name}: step failure {fails}"
        fields = {n: np.empty(config.grid.field_shape) for n in names}
        M = np.empty((3,) + config.grid.cell_shape)
        for r, sl in zip(runs, slabs):
            st = r.save_state()
            c0, c1 = sl.owned_fields
            for n in names:
                fields[n][c0:c1] = parallel.owned_part(sl, st[n])
            M[:, sl.x_lo:sl.x_hi] = parallel.owned_cells(sl, st["M"])
        for k, v in g["fields"].items():
            got = M if k == "M" else fields[k]
            assert np.array_equal(got, v), (name, nranks, k, float(np.max(np.abs(got - v))))
        its = np.asarray(out[0][1], dtype=int) if any_mag else np.zeros(0, dtype=int)
        assert np.array_equal(its, g["iterations"]), (name, nranks, "iterations")
        for p, (comp, loc) in enumerate(keys):
            owner = next(q for q, sl in enumerate(slabs)
                         if sl.owned_fields[0] <= loc[0] < sl.owned_fields[1])
            assert np.array_equal(out[owner][0][:, p], g["probes"][(comp, loc)]), (name, comp, loc)
        cont = int(N.load_library().mpb_continued_steps(runs[0].h))
        return f"OK {name} x{nranks}" + (f" ({cont} continued steps)" if cont else "")
    finally:
        for r in runs:
            r.close()


def _threads(fn, n):
    errs = []

    def go(q):
        try:
            fn(q)
        except Exception as exc:   # reported by the main thread
            errs.append(exc)

    ts = [threading.Thread(target=go, args=(q,)) for q in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


def bench_geometry(cfg_name: str, nranks: int, steps: int, dtype: str = "f64") -> str:
    """bench.py's weak-scaling workload (slab_run: the config's geometry
    repeated along x, one slab per rank, painted tiled materials, a random
    mid-run state) through the NCCL branch, against one handle stepping the
    whole global grid: bit for bit."""
    from pathlib import Path

    import bench
    from paper_2510_22221_b200.config import load_config
    from paper_2510_22221_b200.engine import DeviceRun
    from paper_2510_22221_b200.grid import GridSpec
    from paper_2510_22221_b200.sim import _device_run_args

    cfg = load_config(Path(bench.ROOT) / bench.CONFIGS[cfg_name], lazy=True)
    g = cfg.grid
    ggrid = GridSpec(g.nx * nranks, g.ny, g.nz, g.dx, g.dy, g.dz)
    gcfg = replace(cfg, grid=ggrid, probes=())
    a = _device_run_args(gcfg, [])
    any_mag = cfg.materials.magnetic_count() > 0
    gmats = cfg.materials.tiled_region(0, ggrid.nx)
    state = bench.synthetic_state(ggrid.field_shape, "random")
    m0 = initial_magnetization(gmats)
    src = source_values(cfg.source, cfg.dt, 0, steps)
    kw = {"storage": dtype} if dtype != "f64" else {}
    # fp32 storage has no bitwise contract across step orders (the sweep forms
    # E in fp32, the deferred-E kernel in fp64): the single-handle run then
    # uses the slabs' order (LLG after the sweep); fp64 is the same either way
    if dtype != "f64":
        os.environ["MPB_LLG_PRE"] = "0"
    ref = DeviceRun(ggrid, gmats, a["boundaries"], a["source_loc"], a["source_pol"], [],
                    cfg.llg_params, cfg.dt, device=0, **kw)
    os.environ.pop("MPB_LLG_PRE", None)
    try:
        ref.load_state(state, m0)
        _, _, fail = ref.run(0, src)
        assert fail is None, fail
        want = ref.save_state()
    finally:
        ref.close()
    nid = nccl_id()
    slabs = [replace(s, nccl_id=nid) for s in parallel.make_slabs(ggrid.nx, nranks, any_mag)]
    runs = [DeviceRun(ggrid, cfg.materials.tiled_region(*s.cell_range), a["boundaries"],
                      a["source_loc"], a["source_pol"], [], cfg.llg_params, cfg.dt, device=0,
                      slab=s, **kw) for s in slabs]
    names = ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")
    try:
        for r, sl in zip(runs, slabs):
            r.load_state({n: parallel.local_fields(sl, state[n]) for n in names},
                         parallel.local_cells(sl, m0, axis=1))
        res = [None] * nranks

        def go(q):
            res[q] = runs[q].run(0, src)

        _threads(go, nranks)
        assert all(x[2] is None for x in res), [x[2] for x in res]
        for r, sl in zip(runs, slabs):
            st = r.save_state()
            c0, c1 = sl.owned_fields
            for n in names:
                assert np.array_equal(parallel.owned_part(sl, st[n]), want[n][c0:c1]), (n, c0)
            assert np.array_equal(parallel.owned_cells(sl, st["M"]),
                                  want["M"][:, sl.x_lo:sl.x_hi]), ("M", sl.x_lo)
    finally:
        for r in runs:
            r.close()
    return f"OK bench {cfg_name} {dtype} x{nranks} {steps} steps"


if __name__ == "__main__":
    if sys.argv[1] == "bench":
        print(bench_geometry(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]),
                             sys.argv[5] if len(sys.argv) > 5 else "f64"), flush=True)
        sys.exit(0)
    n = int(sys.argv[1])
    for name in sys.argv[2:]:
        print(run_case(name, n), flush=True)
