"""ctypes binding of the C ABI in ``include/magphon_b200.h``.

The shared library is built in-tree (``csrc/Makefile`` or
``__graft_entry__.build()``) as ``paper_2510_22221_b200/_magphon_b200.so``.
There is no fallback: if the library or a CUDA device is missing, every
entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).with_name("_magphon_b200.so")

OK, EINVAL, ESTEP, ECUDA = 0, 1, 2, 3
FACE_CODES = {"PEC": 0, "PMC": 1, "MUR1": 2}
COMP_CODES = {n: i for i, n in enumerate(
    ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz", "Mx", "My", "Mz"))}
MAX_MATERIALS = 256
MAX_ITERS_CAP = 1000


class Material(C.Structure):
    _fields_ = [("ca", C.c_double), ("cb", C.c_double),
                ("mur_k", C.c_double * 3), ("Ms", C.c_double),
                ("alpha_ms", C.c_double), ("c_llg", C.c_double),
                ("hbias", C.c_double * 3), ("magnetic", C.c_int32),
                ("pad_", C.c_int32), ("eps", C.c_double)]


class Setup(C.Structure):
    _fields_ = [("n", C.c_int32 * 3), ("d", C.c_double * 3),
                ("dt", C.c_double), ("coef_h", C.c_double),
                ("faces", C.c_int32 * 6), ("n_materials", C.c_int32),
                ("materials", C.POINTER(Material)),
                ("cell_material", C.POINTER(C.c_uint8)),
                ("src_loc", C.c_int32 * 3), ("src_pol", C.c_double * 3),
                ("n_probes", C.c_int32),
                ("probe_comp", C.POINTER(C.c_int32)),
                ("probe_loc", C.POINTER(C.c_int32)),
                ("llg_tol", C.c_double), ("llg_max_iters", C.c_int32),
                ("device", C.c_int32), ("kernel_variant", C.c_int32),
                ("graph_steps", C.c_int32),
                ("nranks", C.c_int32), ("rank", C.c_int32),
                ("x_lo", C.c_int32), ("x_hi", C.c_int32),
                ("any_magnetic", C.c_int32), ("nccl_id", C.c_uint8 * 128),
                ("storage", C.c_int32)]


STORAGE_CODES = {"f64": 0, "f32": 1}


class Failure(C.Structure):
    _fields_ = [("step", C.c_int64), ("residual", C.c_double),
                ("iterations", C.c_int32), ("kind", C.c_int32)]


EXPORTS = ("mpb_version", "mpb_last_error", "mpb_nccl_unique_id", "mpb_create", "mpb_destroy",
           "mpb_load_state", "mpb_save_state", "mpb_run", "mpb_run_device",
           "mpb_check_failure", "mpb_set_kernel_timing", "mpb_kernel_time",
           "mpb_launch_count", "mpb_device_bytes", "mpb_selftest_division",
           "mpb_group_run", "mpb_total_energy", "mpb_comm_info", "mpb_sweep_form",
           "mpb_continued_steps", "mpb_hankel_mul")

_lib = None


def load_library(path: os.PathLike | None = None) -> C.CDLL:
    """Load (once) and prototype the shared library; raises if absent."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("MAGPHON_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"magphon_b200 CUDA library not built ({p}); run "
            "`python -c 'import __graft_entry__ as g; g.build()'` or "
            "`make -C paper_2510_22221_b200/csrc`")
    lib = C.CDLL(str(p))
    P = C.POINTER
    dbl_pp = C.POINTER(C.c_double) * 6
    proto = {
        "mpb_version": (C.c_char_p, []),
        "mpb_last_error": (C.c_char_p, []),
        "mpb_nccl_unique_id": (C.c_int, [P(C.c_uint8)]),
        "mpb_create": (C.c_int, [P(Setup), P(C.c_void_p)]),
        "mpb_destroy": (None, [C.c_void_p]),
        "mpb_load_state": (C.c_int, [C.c_void_p, dbl_pp, P(C.c_double)]),
        "mpb_save_state": (C.c_int, [C.c_void_p, dbl_pp, P(C.c_double)]),
        "mpb_run": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, P(C.c_double),
                              P(C.c_double), P(C.c_int32), P(Failure)]),
        "mpb_run_device": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64,
                                     C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p]),
        "mpb_check_failure": (C.c_int, [C.c_void_p, P(Failure)]),
        "mpb_set_kernel_timing": (C.c_int, [C.c_void_p, C.c_int]),
        "mpb_kernel_time": (C.c_int, [C.c_void_p, P(C.c_double), P(C.c_int64),
                                      P(C.c_char_p)]),
        "mpb_launch_count": (C.c_int64, [C.c_void_p]),
        "mpb_device_bytes": (C.c_int64, [C.c_void_p]),
        "mpb_total_energy": (C.c_int, [C.c_void_p, P(C.c_double)]),
        "mpb_continued_steps": (C.c_int64, [C.c_void_p]),
        "mpb_hankel_mul": (C.c_int, [C.c_int32, P(C.c_double), C.c_int64, C.c_int32, C.c_int32,
                                     C.c_int32, P(C.c_double), P(C.c_double)]),
        "mpb_sweep_form": (C.c_int, [C.c_void_p, P(C.c_int32)]),
        "mpb_comm_info": (C.c_int, [C.c_void_p, P(C.c_int32), P(C.c_int32), P(C.c_int32)]),
        "mpb_selftest_division": (C.c_int, [C.c_int32, C.c_double, P(C.c_double),
                                            C.c_int64, P(C.c_int64), P(C.c_double)]),
        "mpb_group_run": (C.c_int, [P(C.c_void_p), C.c_int32, C.c_int64, C.c_int64,
                                    P(C.c_double), P(P(C.c_double)), P(C.c_int32),
                                    P(Failure)]),
    }
    for name, (res, args) in proto.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


def last_error() -> str:
    return load_library().mpb_last_error().decode(errors="replace")


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


def check(code: int) -> None:
    if code != OK:
        msg = last_error()
        if code == EINVAL:
            raise ValueError(msg)
        raise NativeError(code, msg)
