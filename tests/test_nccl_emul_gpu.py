"""The library's real multi-rank code path on one GPU: handles created with
an NCCL id run the NCCL branch of every step (exchange() send/recv pairing
on the split exchange communicator, the in-place all-reduces of the LLG
statistics, the host-continued non-monotone step), with the NCCL entry
points replaced by an in-process emulation (tests/nccl_emul/nccl_emul.cu,
LD_PRELOAD) and one host thread per rank -- bit for bit against the
reference goldens, overlapped and serialised exchange.  (NCCL itself needs
one GPU per rank: tests/test_nccl_gpu.py.)"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "nccl_emul" / "nccl_emul.cu"
LIB = ROOT / "tests" / "nccl_emul" / "libnccl_emul.so"

SPLITS = [(2, ["mixed3d", "allmur3d", "bias3d", "two_magnets", "nonmono3d", "fail3d"]),
          (3, ["mixed3d", "zwall_magnet", "cpw_small", "thin", "nonmono3d"]),
          (4, ["pec_block", "two_magnets", "plane2d"])]


def _shim() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                        "-Xcompiler", "-fPIC", "-o", str(LIB), str(SRC)], check=True)
    return LIB


@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("nranks,cases", SPLITS)
def test_nccl_code_path_matches_reference_goldens(nranks, cases, overlap):
    env = dict(os.environ, LD_PRELOAD=str(_shim()), MPB_OVERLAP=overlap,
               MPB_SWEEP_MINCHUNK="2")
    out = subprocess.run([sys.executable, str(ROOT / "tests" / "nccl_emul_worker.py"),
                          str(nranks)] + cases, cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    for name in cases:
        assert any(line.startswith(f"OK {name} x{nranks}") for line in out.stdout.splitlines()), \
            (name, out.stdout)


# bench.py's weak-scaling workload itself (slab_run geometry: the config
# repeated along x, one slab per rank) through the NCCL branch vs one handle
# stepping the whole global grid
@pytest.mark.parametrize("cfg,nranks,steps,dtype", [("c2", 2, 6, "f64"), ("c3", 2, 4, "f64"),
                                                     ("c2", 3, 4, "f32")])
def test_nccl_code_path_bench_geometry(cfg, nranks, steps, dtype):
    env = dict(os.environ, LD_PRELOAD=str(_shim()), MPB_SWEEP_MINCHUNK="2")
    out = subprocess.run([sys.executable, str(ROOT / "tests" / "nccl_emul_worker.py"), "bench",
                          cfg, str(nranks), str(steps), dtype], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert f"OK bench {cfg} {dtype} x{nranks}" in out.stdout, out.stdout
