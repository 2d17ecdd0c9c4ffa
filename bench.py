#!/usr/bin/env python3
"""Throughput of the coupled Maxwell-LLG step on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4]
    python bench.py --impl reference ...     # CPU reference arm

Workload: C4 of SURVEY 8d -- 1024x1024x128 cells per GPU (CPW line on a Si
substrate + YIG film, all-MUR1 walls, fp64), the per-GPU configuration the
weak-scaling metric is quoted on.  A "step" is one full coupled step
(curl E, H + LLG fixed point, curl H, E, walls, source, probes) of that grid.
`--config c5 [--scaling strong]`: the fixed 2048x2048x256 grid (BASELINE
configs[4]) split over the N GPUs (110 GB of device state on one B200).

Prints ONE JSON line on rank 0:
  value  -- Gcell-updates/s over all ranks, state resident in HBM, device
            timed with CUDA events on the launching stream, max over ranks;
  e2e    -- same metric through the C-ABI call mpb_run with HOST buffers
            (per-step source values H2D, probes + r* D2H inside the timing);
  roofline -- dominant kernel's algorithmic bytes / its event-timed duration
            vs the measured HBM copy bandwidth (MEASURED_PEAKS.json);
  cpu_baseline -- the numpy oracle (restatement of the reference) timed on a
            bounded sample on this host.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {"c1": "configs/c1.cfg", "c2": "configs/c2.cfg", "c3": "configs/c3.cfg",
           "c4": "configs/c4.cfg", "c5": "configs/c5.cfg"}
DESCRIPTIONS = {
    "c1": "vacuum PEC cavity + YIG block, 1000 Oe bias",
    "c2": "CPW resonator on Si + YIG film, all-MUR1",
    "c3": "standalone YIG film on Si, all-MUR1",
    "c4": "CPW line on Si + YIG film, all-MUR1",
    "c5": "CPW line on Si + YIG film, all-MUR1",
}
FALLBACK_HBM = 6650.0
METRIC = "coupled Maxwell-LLG Gcell-updates/s"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


def _bytes_per_cell(f_mag: float, dtype: str = "f64") -> float:
    # 6 field comps read+written once (96 B fp64, 48 B fp32) + M
    # read+write (48 B; M is fp64 in both storage modes) in the magnetic
    # fraction.  Ids/halos/probes are not credited.
    return _sweep_bytes(dtype) + 48.0 * f_mag


def _sweep_bytes(dtype: str) -> float:
    # The dominant kernel (k_sweep) moves the six field components; M is read
    # and written by k_llg_local, so the sweep's algorithmic bytes are 96
    # B/cell (48 B/cell in the fp32 storage mode).
    return 96.0 if dtype == "f64" else 48.0


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, timestamped; summary() keeps the
    samples that fall inside [t0, t1] (the timed region)."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = ""

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0: float, t1: float):
        import datetime
        rows = []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        for line in self.out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                rows.append((ts, float(f[1]), float(f[2]), float(f[3]),
                             [n for n, v in zip(names, f[5:9]) if v.lower() == "active"]))
            except ValueError:
                continue
        if not rows:
            return None
        inside = [r for r in rows if t0 - 0.05 <= r[0] <= t1 + 0.05]
        if not inside:   # short region: the sample closest to its middle
            mid = 0.5 * (t0 + t1)
            inside = [min(rows, key=lambda r: abs(r[0] - mid))]
        reasons = sorted({n for r in inside for n in r[4]})
        return {"sm_mhz": statistics.median(r[1] for r in inside),
                "sm_max_mhz": max(r[2] for r in rows),
                "power_w_max": max(r[3] for r in inside),
                "reasons": reasons, "samples": len(inside)}


def synthetic_state(fs, kind: str):
    """Initial E, H for the benchmark.

    "random": a mid-run-like state -- every entry carries a nonzero field
    (E ~ 1e3 V/m, H ~ E/377), so no arithmetic is skipped or degenerate (a
    fresh run is exact zeros almost everywhere for thousands of steps).
    "zero": the reference's own initial state.
    """
    fs = tuple(fs)
    if kind == "zero":
        z = np.zeros(fs)
        return {n: z for n in ("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")}
    rng = np.random.default_rng(1234)
    base = rng.standard_normal(fs)
    out = {}
    for q, n in enumerate(("Ex", "Ey", "Ez", "Hx", "Hy", "Hz")):
        scale = 1e3 * (1.0 + 0.1 * q) if n[0] == "E" else 2.65 * (1.0 + 0.1 * q)
        out[n] = np.roll(base, q, axis=-1)
        out[n] *= scale                      # in place: C5 fields are 8.6 GB each
    return out


def _device_class():
    """engine.DeviceRun, or (tests only) the class named by MPB_BENCH_DEVICE
    as "module:Class" -- lets a CPU test drive the multi-rank set-up."""
    spec = os.environ.get("MPB_BENCH_DEVICE")
    if spec:
        import importlib
        mod, cls = spec.split(":")
        return getattr(importlib.import_module(mod), cls)
    from paper_2510_22221_b200.engine import DeviceRun
    return DeviceRun


def slab_run(cfg, keys, world, rank, local, args, nccl: bool = True):
    """One rank's x-slab, NCCL exchange with its neighbours.

    weak (C4, BASELINE configs[3]): the global grid is the config's geometry
    repeated along x, (nx * world) x ny x nz; rank r owns [nx r, nx (r+1));
    source on rank 0's slab, no probes.
    strong (C5, configs[4]): the config's own grid split into `world` slabs;
    source and probes where the config puts them.
    Materials stay painted (lazy): each rank builds only its slab's ids."""
    import torch.distributed as dist
    from dataclasses import replace

    from paper_2510_22221_b200 import parallel
    from paper_2510_22221_b200.grid import GridSpec, initial_magnetization
    from paper_2510_22221_b200.sim import _device_run_args

    g = cfg.grid
    nccl_id = parallel.nccl_unique_id(dist) if world > 1 and nccl else bytes(128)
    if args.scaling == "weak":
        ggrid = GridSpec(g.nx * world, g.ny, g.nz, g.dx, g.dy, g.dz)
        gcfg = replace(cfg, grid=ggrid, probes=())
        keys = []
    else:
        ggrid, gcfg = g, cfg
    any_mag = cfg.materials.magnetic_count() > 0
    slab = replace(parallel.make_slabs(ggrid.nx, world, any_mag)[rank], nccl_id=nccl_id)
    c0, c1 = slab.cell_range
    mats = (cfg.materials.tiled_region(c0, c1) if args.scaling == "weak"
            else cfg.materials.region(c0, c1))
    a = _device_run_args(gcfg, keys)
    dev = _device_class()(ggrid, mats, a["boundaries"], a["source_loc"], a["source_pol"], keys,
                          cfg.llg_params, cfg.dt, device=local, kernel_variant=args.variant,
                          slab=slab, **({"storage": args.dtype}
                                        if getattr(args, "dtype", "f64") != "f64" else {}))
    f0, f1 = slab.field_range
    st = synthetic_state((f1 - f0,) + tuple(ggrid.field_shape[1:]), args.init)
    dev.load_state(st, initial_magnetization(mats))
    del st
    return dev, (slab.x_hi - slab.x_lo) * g.ny * g.nz


def slab_sample_config(cfg, x0: int, x1: int):
    """The config's cell planes [x0, x1) as a stand-alone config for the CPU
    reference: same y-z geometry, materials and walls, the source only if it
    lies in the slab (else a zero-amplitude one), no probes.  Per-cell work is that of the whole grid."""
    from dataclasses import replace

    from paper_2510_22221_b200 import em
    from paper_2510_22221_b200.grid import GridSpec
    g = cfg.grid
    sub = GridSpec(x1 - x0, g.ny, g.nz, g.dx, g.dy, g.dz)
    mats = cfg.materials.region(x0, x1)
    src = cfg.source
    loc = src.location
    if x0 <= loc[0] < x1:
        src = replace(src, location=(loc[0] - x0, loc[1], loc[2]))
    else:                        # same per-step work, nothing injected
        src = replace(src, location=(0, loc[1], loc[2]), amplitude=0.0)
    return replace(cfg, grid=sub, materials=mats, source=src, probes=())


def _oracle_steps(cfg, warm: int, steps: int):
    """Run the numpy oracle for warm + steps steps; returns the seconds of the
    last `steps` (set-up and warm-up excluded)."""
    from oracle import magphon_oracle as orc
    marks = []
    orc.run(cfg, n_steps=warm + steps, marks=marks)
    return marks[-1] - marks[warm]


def cpu_oracle_sample(cfg_name: str, planes: int, steps: int):
    """Time the numpy oracle (restatement of the reference CPU path) on one
    host core over the first `planes` x-planes of the bench config; returns
    (Gcell-updates/s, seconds, cells)."""
    from paper_2510_22221_b200.config import load_config
    cfg = load_config(ROOT / CONFIGS[cfg_name], lazy=True)
    planes = max(2, min(planes, cfg.grid.nx))
    sub = slab_sample_config(cfg, 0, planes)
    cells = int(np.prod(sub.grid.cell_shape))
    secs = _oracle_steps(sub, 1, steps)
    return cells * steps / secs / 1e9, secs, cells


def _replica_worker(cfg_name, x0, x1, warm, steps, barrier, out):
    """One replica of the reference arm: its x-slab of the bench config."""
    from paper_2510_22221_b200.config import load_config
    cfg = slab_sample_config(load_config(ROOT / CONFIGS[cfg_name], lazy=True), x0, x1)
    cfg.materials.Ms                          # dense maps before the start line
    barrier.wait()
    out.put(_oracle_steps(cfg, warm, steps))


def cpu_slab_replicas(cfg_name: str, slabs, warm: int, steps: int):
    """The reference's CPU path on all host cores at once: one single-threaded
    oracle process per x-slab (the reference's numpy ufuncs are single
    threaded; its own parallelism is a process pool, sim.py:243-260).
    Returns (aggregate Gcell-updates/s, slowest replica's seconds, cells)."""
    import multiprocessing as mp

    from paper_2510_22221_b200.config import load_config
    g = load_config(ROOT / CONFIGS[cfg_name], lazy=True).grid
    cells = sum(x1 - x0 for x0, x1 in slabs) * g.ny * g.nz
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(len(slabs))
    out = ctx.Queue()
    ps = [ctx.Process(target=_replica_worker, args=(cfg_name, x0, x1, warm, steps, barrier, out))
          for x0, x1 in slabs]
    for p in ps:
        p.start()
    secs = [out.get() for _ in ps]
    for p in ps:
        p.join()
    worst = max(secs)
    return cells * steps / worst / 1e9, worst, cells


def reference_slabs(nx: int, ny: int, nz: int, cores: int, max_planes: int | None = None):
    """x-slabs of [0, nx) for `cores` replicas, at most ~300 B/cell of half the
    available host memory in total (the oracle's dense arrays)."""
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except ImportError:
        avail = 16 << 30
    budget = int(0.5 * avail // (300 * ny * nz))           # planes that fit
    planes = min(nx, budget)
    if max_planes is not None:
        planes = min(planes, max_planes * cores)
    cores = max(1, min(cores, planes // 2))
    per = max(2, planes // cores)
    return [(r * per, (r + 1) * per) for r in range(cores)]


def run_reference(args) -> None:
    """Reference arm: the reference's CPU path (the numpy oracle port; the
    reference package cannot travel to the GPU box) on all usable host cores,
    on the GPU arm's own workload: the bench config's x-planes split into one
    slab per core (the whole grid when host memory allows), every replica
    stepping its slab concurrently.  Under torchrun only rank 0 runs."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2510_22221_b200.config import load_config
    cfg = load_config(ROOT / CONFIGS[args.config], lazy=True)
    g = cfg.grid
    cores = len(os.sched_getaffinity(0))
    slabs = reference_slabs(g.nx, g.ny, g.nz, cores, args.ref_planes)
    # one untimed step sizes the sample so that W + K steps stay within ~3 min
    _, one, _ = cpu_slab_replicas(args.config, slabs, 0, 1)
    budget = 180.0 / max(1, args.steps + args.warmup)
    while one > budget and slabs[0][1] - slabs[0][0] > 2:
        per = max(2, (slabs[0][1] - slabs[0][0]) // 2)
        slabs = [(r * per, (r + 1) * per) for r in range(len(slabs))]
        one /= 2.0
    v, secs, cells = cpu_slab_replicas(args.config, slabs, args.warmup, args.steps)
    world = max(1, args.gpus)
    total_cells = int(np.prod(g.cell_shape)) * (world if args.scaling == "weak" else 1)
    line = {
        "metric": METRIC, "value": v, "unit": "Gcell-updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": workload_config(args, cfg, world, total_cells),
        "cpu_baseline": {
            "value": v, "unit": "Gcell-updates/s", "cores": len(slabs), "kind": "port",
            "sample": f"numpy oracle (restatement of magphon.sim.run, one thread per "
                      f"process like the reference) on {len(slabs)} host cores at once, "
                      f"each stepping an x-slab of {slabs[0][1] - slabs[0][0]} planes of "
                      f"{args.config.upper()} ({cells} of its {int(np.prod(g.cell_shape))} "
                      f"cells per step), {args.warmup} + {args.steps} steps, slowest "
                      f"replica {secs:.1f} s; per-cell CPU cost does not depend on N"},
        "e2e": {"value": v, "unit": "Gcell-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _l2_note(g, dtype: str) -> str:
    """Whether the per-GPU state is larger than the 126 MB L2 (no flush is
    needed between steps) or resident in it (small configs)."""
    entries = (g.nx + 1) * (g.ny + 1) * (g.nz + 1)
    state = 2 * 6 * entries * (8 if dtype == "f64" else 4)
    mb = state / 1e6
    if state > 2 * 126e6:
        return f"state (2 x 6 field arrays, {mb:.0f} MB) >> 126 MB L2; no flush needed"
    return (f"state (2 x 6 field arrays, {mb:.0f} MB) is L2-resident between steps, as in "
            f"any run of this size; not flushed")


def workload_config(args, cfg, world: int, total_cells: int) -> dict:
    """The `config` object of the JSON line (identical in both arms)."""
    g = cfg.grid
    cells = int(np.prod(g.cell_shape))
    per_gpu = cells if args.scaling == "weak" else cells // max(1, world)
    return {"workload": f"{args.config.upper()} {'x'.join(map(str, g.cell_shape))} "
                        + ("cells per GPU" if args.scaling == "weak" else
                           f"cells split over {world} GPU(s)")
                        + f", {DESCRIPTIONS[args.config]}, "
                        + ("fp64" if getattr(args, "dtype", "f64") == "f64"
                           else "fp32 E/H storage (M + LLG fp64)"),
            "config_file": CONFIGS[args.config], "cells_per_gpu": per_gpu,
            "cells_total": total_cells,
            "magnetic_fraction": cfg.materials.magnetic_count() / cells,
            "parallelism": f"x-slab x{world}" if world > 1 else "single GPU",
            "l2": _l2_note(g, getattr(args, "dtype", "f64")),
            "kernel_variant": args.variant,
            "initial_state": args.init}


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(nproc: int) -> int:
    """`python bench.py --gpus N` without torchrun: re-run this command as N
    ranks under torch.distributed.run (one process per GPU, rendezvous on
    127.0.0.1), the launch the multi-GPU driver uses."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    print(f"[bench] launching {nproc} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, cwd=str(ROOT))


def layout_only(args, world: int, rank: int) -> None:
    """(test hook) build this rank's slab exactly as the timed run would and
    record it as JSON in args.layout_only; no device work, gloo plumbing."""
    import torch.distributed as dist

    from paper_2510_22221_b200.config import load_config
    dist.init_process_group("gloo")
    cfg = load_config(ROOT / CONFIGS[args.config], lazy=True)
    keys = list(dict.fromkeys((p[0], (p[1], p[2], p[3])) for p in cfg.probes))
    dev, cells = slab_run(cfg, keys, world, rank, 0, args, nccl=False)
    sl = dev.slab
    rec = {"rank": rank, "world": world, "env_world": int(os.environ["WORLD_SIZE"]),
           "x_lo": sl.x_lo, "x_hi": sl.x_hi, "nranks": sl.nranks, "cells": cells,
           "grid": list(dev.grid.cell_shape)}
    Path(args.layout_only, f"rank{rank}.json").write_text(json.dumps(rec))
    dist.barrier()
    dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"],
                    help="field storage: f64 (reference precision, bit-exact; the "
                         "headline) or f32 (opt-in, E/H in fp32, M + LLG in fp64)")
    ap.add_argument("--cpu-planes", type=int, default=32,
                    help="x-planes of the bench config in the 1-core cpu_baseline sample")
    ap.add_argument("--cpu-steps", type=int, default=8)
    ap.add_argument("--ref-planes", type=int, default=None,
                    help="reference arm: at most this many x-planes per host core")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--init", default="random", choices=["random", "zero"])
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="multi-GPU mode (default: weak for c1-c4, strong for c5)")
    ap.add_argument("--layout-only", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the C3 fp64 and C4 fp32 secondary records of the default run")
    args = ap.parse_args()
    if args.scaling is None:
        args.scaling = "strong" if args.config == "c5" else "weak"
    if args.impl == "reference":
        run_reference(args)
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch "
                         f"with --nproc-per-node {args.gpus} or without torchrun")
    if args.layout_only:
        layout_only(args, world, rank)
        return
    if world > 1:
        # a rank stuck in a collective (a peer died, a mis-paired exchange)
        # ends the run with every thread's stack instead of hanging the job
        import faulthandler
        faulthandler.dump_traceback_later(int(os.environ.get("MPB_BENCH_WATCHDOG_S", "1200")),
                                          exit=True)

    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    line = measure(args, world, rank, local)
    if line is None:
        return
    if world == 1 and not args.no_secondary and args.config == "c4" and args.dtype == "f64":
        # secondary records measured by this same run: the LLG-heavy config
        # (C3: 7% magnetic cells) and the fp32 storage mode on the headline grid
        line["secondary"] = []
        for cfg_name, dtype in (("c3", "f64"), ("c4", "f32")):
            sub = argparse.Namespace(**vars(args))
            sub.config, sub.dtype, sub.no_cpu = cfg_name, dtype, True
            sub.scaling = "weak"
            sub.steps, sub.warmup = max(20, args.steps), max(3, args.warmup)
            sl = measure(sub, world, rank, local)
            line["secondary"].append({
                "workload": sl["config"]["workload"], "dtype": dtype,
                "value": sl["value"], "unit": sl["unit"], "e2e": sl["e2e"]["value"],
                "ms_per_step": sl["ms_per_step"], "steps": sl["steps"],
                "roofline_frac": sl["roofline"]["frac"],
                "whole_step_frac": sl["roofline"]["whole_step_frac"],
                "bytes_per_cell": sl["roofline"]["bytes_per_cell"],
                "magnetic_fraction": sl["config"]["magnetic_fraction"],
                "clocks": sl["clocks"], "gpu_launches": sl["gpu_launches"]})
    print(json.dumps(line))


def measure(args, world, rank, local):
    """One bench measurement (timed device region, e2e leg, roofline, CPU
    baseline unless --no-cpu); returns the JSON line on rank 0, else None."""
    import torch

    from paper_2510_22221_b200 import sim
    from paper_2510_22221_b200.config import load_config
    from paper_2510_22221_b200.grid import initial_magnetization

    # painted (lazy) materials: no dense per-cell host maps (C5 would need 69 GB)
    cfg = load_config(ROOT / CONFIGS[args.config], lazy=True)
    cells = int(np.prod(cfg.grid.cell_shape))        # per GPU (weak) / total (strong)
    mag = cfg.materials.magnetic_count()
    f_mag = mag / cells
    keys = [(p[0], (p[1], p[2], p[3])) for p in cfg.probes]
    keys = list(dict.fromkeys(keys))
    if world == 1:
        dev = sim._device_run(cfg, cfg.materials, keys, device=local,
                              kernel_variant=args.variant, storage=args.dtype)
        dev.load_state(synthetic_state(cfg.grid.field_shape, args.init),
                       initial_magnetization(cfg.materials))
        rank_cells = cells
    else:
        dev, rank_cells = slab_run(cfg, keys, world, rank, local, args)
    total_cells = cells * world if args.scaling == "weak" else cells
    gwarm = 32                        # untimed: instantiates the 16-step CUDA graph
    total = args.warmup + gwarm + 2 * args.steps
    src = torch.tensor(sim.source_values(cfg.source, cfg.dt, 0, total),
                       dtype=torch.float64, device="cuda")
    probe = torch.zeros((total, max(1, len(keys))), dtype=torch.float64, device="cuda")
    iters = torch.zeros(total, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def run(n0, n):
        dev.run_device(n0, n, src[n0:].data_ptr(), probe[n0:].data_ptr(), iters[n0:].data_ptr(),
                       stream.cuda_stream)

    def timed(n0, n):
        """K steps between a barrier + synchronize on both sides, CUDA events
        on the launching stream; max over ranks."""
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(n0, n)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        t = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([t], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            t = float(tt.item())
        return t

    # warm-up: W untimed steps, then the graph instantiation (untimed)
    run(0, args.warmup)
    run(args.warmup, gwarm)
    torch.cuda.synchronize()
    if dev.check_failure() is not None:
        raise RuntimeError("LLG failure during warm-up")
    n0 = args.warmup + gwarm
    clk = ClockSampler(local).start()
    t_wall0 = time.time()
    # timed region 1 -> value: K steps, device-resident state, the product
    # path (16-step CUDA graphs)
    ms = timed(n0, args.steps)
    launches = dev.launch_count()
    # timed region 2 -> roofline: the next K steps with CUDA events around
    # every launch of the dominant kernel on its own (library) stream; the
    # per-kernel events disable the graphs, so this region's step time is
    # reported next to the kernel's for the kernel share
    dev.set_kernel_timing(True)
    ms_k = timed(n0 + args.steps, args.steps)
    t_wall1 = time.time()
    clk.stop()
    kms, klaunch, kname = dev.kernel_time()
    dev.set_kernel_timing(False)
    fail = dev.check_failure()
    if fail is not None:
        raise RuntimeError(f"LLG failure in timed region: {fail}")
    value = total_cells * args.steps / (ms * 1e-3) / 1e9
    # end-to-end through the C ABI with host buffers (mpb_run)
    e2e_steps = args.e2e_steps or args.steps
    # untimed warm-up of the host-buffer path (allocates its staging buffers)
    warm = 32
    _, _, fail = dev.run(total, sim.source_values(cfg.source, cfg.dt, total, total + warm))
    if fail is not None:
        raise RuntimeError(f"LLG failure in e2e warm-up: {fail}")
    total += warm
    # inputs and results in pinned host memory (page-locked, like a
    # production pipeline's staging buffers)
    pin_src = torch.from_numpy(
        sim.source_values(cfg.source, cfg.dt, total, total + e2e_steps)).pin_memory()
    pin_probe = torch.zeros((e2e_steps, max(1, len(dev.probes))),
                            dtype=torch.float64).pin_memory()
    pin_iters = torch.zeros(e2e_steps, dtype=torch.int32).pin_memory()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, _, fail = dev.run(total, pin_src.numpy(), pin_probe.numpy(), pin_iters.numpy())
    t_e2e = time.perf_counter() - t0
    if fail is not None:
        raise RuntimeError(f"LLG failure in the e2e leg: {fail}")
    if world > 1:
        t = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(t.item())
    e2e = total_cells * e2e_steps / t_e2e / 1e9
    peak, peak_kind = _peaks()
    bpc = _sweep_bytes(args.dtype) if kname == "k_sweep" else _bytes_per_cell(f_mag, args.dtype)
    per_launch_ms = kms / max(1, klaunch)
    achieved = rank_cells * bpc / (per_launch_ms * 1e-3) / 1e9 if klaunch else None
    step_frac = value / world * _bytes_per_cell(f_mag, args.dtype) / peak   # per-GPU average
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists() and args.config == "c4" and world == 1:   # captured on C4, 1 GPU
        traffic = json.loads(tp.read_text()).get(kname if args.dtype == "f64"
                                                 else f"{kname}_{args.dtype}")
    comm = dev.comm_info()
    if world > 1:
        gathered = [None] * world
        torch.distributed.all_gather_object(gathered, comm)
        comm = {"nranks_per_comm": sorted({c["nranks"] for c in gathered}),
                "ranks": [c["rank"] for c in gathered],
                "nccl_version": comm["nccl_version"]}
    if rank != 0:
        dev.close()
        return
    cpu = None
    if not args.no_cpu:
        rate, secs, ccells = cpu_oracle_sample(args.config, args.cpu_planes, args.cpu_steps)
        cpu = {"value": rate, "unit": "Gcell-updates/s", "cores": 1, "kind": "port",
               "sample": f"numpy oracle (restatement of magphon.sim.run, single "
                         f"thread like the reference) on the first {args.cpu_planes} "
                         f"x-planes of {args.config.upper()} ({ccells} cells) x "
                         f"{args.cpu_steps} steps = {secs:.1f} s"}
    line = {
        "metric": METRIC, "value": value, "unit": "Gcell-updates/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic",
        "config": workload_config(args, cfg, world, total_cells),
        "e2e": {"value": e2e, "unit": "Gcell-updates/s",
                "h2d_bytes_per_step": 8, "d2h_bytes_per_step": 8 * len(dev.probes) + 4,
                "api": "mpb_run (pinned host source values in, pinned host probes + r* out)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak if achieved else None,
                     "traffic": traffic, "kernel": kname,
                     "bytes_per_cell": bpc, "peak_kind": peak_kind,
                     "kernel_ms_per_step": per_launch_ms,
                     "kernel_share_of_step": per_launch_ms / (ms_k / args.steps),
                     "kernel_timing": "CUDA events around each launch on the library "
                                      "stream, in a second timed region of K steps "
                                      f"({ms_k / args.steps:.4f} ms/step there: per-kernel "
                                      "events disable the CUDA graphs of the first)",
                     "whole_step_frac": step_frac,
                     "whole_step_bytes_per_cell": _bytes_per_cell(f_mag, args.dtype)},
        "cpu_baseline": cpu,
        "clocks": clk.summary(t_wall0, t_wall1),
        "gpu_launches": launches,
        "ranks": comm,
    }
    dev.close()
    return line


if __name__ == "__main__":
    main()
