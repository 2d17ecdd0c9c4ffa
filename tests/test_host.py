"""Host-side logic: ABI exports, config schema, material table, sources."""

import ctypes as C
import math
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2510_22221_b200 import _native, em, sim
from paper_2510_22221_b200.config import ConfigError, load_config, parse_quantity
from paper_2510_22221_b200.constants import CONSTANTS, oersted_to_si
from paper_2510_22221_b200.engine import material_table
from tests.golden.cases import CASES, build, mirror_namespace

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_every_header_symbol():
    header = (ROOT / "include" / "magphon_b200.h").read_text()
    declared = set(re.findall(r"\b(mpb_[a-z_]+)\s*\(", header))
    assert declared == set(_native.EXPORTS)
    lib = _native.load_library()
    for name in declared:
        assert getattr(lib, name) is not None
    assert b"sm_100a" in lib.mpb_version()


def test_struct_layout_matches_header():
    # offsets the C side relies on (x86-64 SysV)
    assert C.sizeof(_native.Material) == 11 * 8 + 8 + 8
    assert _native.Setup.dt.offset == 40


def test_create_rejects_invalid_setup():
    lib = _native.load_library()
    su = _native.Setup()
    h = C.c_void_p()
    assert lib.mpb_create(C.byref(su), C.byref(h)) == _native.EINVAL
    assert "cell counts" in _native.last_error()


def test_parse_quantity_units():
    assert parse_quantity("5 um") == 5 * 1e-6
    assert parse_quantity("2050 Oe") == oersted_to_si(2050.0)
    assert parse_quantity("0.003") == 0.003
    with pytest.raises(ValueError):
        parse_quantity("3 furlongs")


CFG = """
[grid]
nx = 8
ny = 6
nz = 4
dx = 10 um
dy = 10 um
dz = 2 um
[background]
eps_r = 2.0
[material:a]
box = 1 3 1 3 1 2
Ms = 1750 G
alpha = 1e-3
bias = 1000 Oe
bias_direction = 0 1 0
[source]
f0 = 15 GHz
Tp = 20 ps
location = 2 2 1
[boundaries]
x0 = MUR1
z1 = PMC
[run]
t_end = 0.3 ps
[probes]
p = Ex 1 1 1
m = Mz 1 1 1
[sweep]
bias_list = 900 Oe, 1000 Oe
"""


def test_load_config_schema(tmp_path):
    p = tmp_path / "c.cfg"
    p.write_text(CFG)
    cfg = load_config(p)
    assert cfg.grid.cell_shape == (8, 6, 4)
    assert cfg.boundaries.x0 == "MUR1" and cfg.boundaries.y0 == "PEC"
    assert cfg.materials.Ms[1, 1, 1] == 1750 * 1000 / (4 * math.pi)
    assert cfg.bias_sweep == (oersted_to_si(900.0), oersted_to_si(1000.0))
    assert cfg.llg_params.tol == 1e-6 and cfg.llg_params.max_iters == 50
    bad = CFG.replace("box = 1 3 1 3 1 2", "box = 1 3 1 3 1")
    p.write_text(bad)
    with pytest.raises(ConfigError):
        load_config(p)
    p.write_text(CFG.replace("x0 = MUR1", "x0 = ABC"))
    with pytest.raises(ConfigError):
        load_config(p)


def test_material_table_reproduces_reference_coefficients():
    cfg = build(CASES["mixed3d"], mirror_namespace())
    dt = cfg.dt
    ids, table = material_table(cfg.materials, dt, cfg.grid.spacings)
    m = cfg.materials
    eps = CONSTANTS.eps0 * m.eps_r
    ca = 1.0 / (m.sigma / 2.0 + eps / dt)
    cb = m.sigma / 2.0 - eps / dt
    got_ca = np.array([table[i].ca for i in range(len(table))])[ids]
    got_cb = np.array([table[i].cb for i in range(len(table))])[ids]
    assert np.array_equal(got_ca, ca) and np.array_equal(got_cb, cb)
    mag = m.Ms > 0
    got_mag = np.array([table[i].magnetic for i in range(len(table))])[ids]
    assert np.array_equal(got_mag.astype(bool), mag)
    c = CONSTANTS.mu0 * np.abs(m.gamma_e) * dt / 2.0
    got_c = np.array([table[i].c_llg for i in range(len(table))])[ids]
    assert np.array_equal(got_c[mag], c[mag])
    for a in range(3):
        cl = 1.0 / np.sqrt(CONSTANTS.mu0 * eps)
        k = (cl * dt - cfg.grid.spacings[a]) / (cl * dt + cfg.grid.spacings[a])
        got_k = np.array([table[i].mur_k[a] for i in range(len(table))])[ids]
        assert np.array_equal(got_k, k)


def test_source_values_bitwise():
    src = em.SourceSpec(f0=14.3e9, Tp=50e-12, amplitude=1e3)
    dt = 6.0042e-15
    vals = sim.source_values(src, dt, 3, 50)
    for n, v in zip(range(3, 50), vals):
        t = (n + 1) * dt
        env = math.exp(-((t - 3.0 * src.Tp) ** 2) / (2.0 * src.Tp ** 2))
        assert v == src.amplitude * env * math.cos(2.0 * math.pi * src.f0 * t)


def test_simconfig_validation():
    cfg = build(CASES["small1d_strong"], mirror_namespace())
    with pytest.raises(ValueError):
        sim.SimConfig(**{**cfg.__dict__, "probes": (("Ex", 0, 0, 10_000),)})
    with pytest.raises(ValueError):
        sim.SimConfig(**{**cfg.__dict__, "t_end": 0.0})


def test_nccl_emulation_covers_every_nccl_import(tmp_path):
    """tests/nccl_emul (the in-process NCCL the multi-rank GPU tests preload)
    builds for sm_100a and defines every NCCL function the library imports."""
    import shutil
    import subprocess
    if not shutil.which("nvcc") or not shutil.which("nm"):
        pytest.skip("needs nvcc and nm")
    lib = _native.LIB_PATH
    out = tmp_path / "libnccl_emul.so"
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                    "-Xcompiler", "-fPIC", "-o", str(out),
                    str(ROOT / "tests" / "nccl_emul" / "nccl_emul.cu")], check=True)

    def syms(path, kind):
        text = subprocess.run(["nm", "-D", str(path)], capture_output=True, text=True).stdout
        return {ln.split()[-1] for ln in text.splitlines()
                if ln.split()[-2:-1] == [kind] and ln.split()[-1].startswith("nccl")}

    imported = syms(lib, "U")
    assert "ncclSend" in imported and "ncclAllReduce" in imported
    assert imported <= syms(out, "T"), imported - syms(out, "T")
