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


if __name__ == "__main__":
    n = int(sys.argv[1])
    for name in sys.argv[2:]:
        print(run_case(name, n), flush=True)
