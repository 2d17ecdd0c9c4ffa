"""Command-line entry point for the GPU path (reference ``cli.py``).

``simulate`` and ``sweep`` keep the reference's flags, output files (probe
text files with the same header and ``%.12e`` values, ``spectrum_map.txt``,
``manifest.json`` with sha256 digests) and exit codes (0 ok, 1 usage/config
error, 2 runtime failure incl. StepFailure).  The reference's other
subcommands (oracle, curate, train, predict) are outside the stepping hot
path and stay in ``magphon``.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

from . import __version__, sim
from .config import ConfigError, load_config, parse_quantity
from .llg import StepFailure

EXIT_OK, EXIT_USAGE, EXIT_RUNTIME = 0, 1, 2
_FMT = "%.12e"


def _sha256(path: Path) -> str:
    h = hashlib.sha256()
    with open(path, "rb") as f:
        for chunk in iter(lambda: f.read(1 << 20), b""):
            h.update(chunk)
    return h.hexdigest()


def _manifest(out: Path, command: str, cfg_path, files, started, diagnostics) -> None:
    doc = {"command": command, "engine_version": __version__, "config": cfg_path,
           "config_sha256": _sha256(Path(cfg_path)) if cfg_path else None,
           "started_unix": started, "finished_unix": time.time(),
           "outputs": [{"path": str(p.relative_to(out)), "sha256": _sha256(p)}
                       for p in files],
           "diagnostics": diagnostics}
    (out / "manifest.json").write_text(json.dumps(doc, indent=2, sort_keys=True) + "\n")


def _out_dir(args) -> Path:
    out = Path(args.out or os.environ.get("MAGPHON_OUT", "."))
    out.mkdir(parents=True, exist_ok=True)
    return out


def write_probe(path: Path, series) -> None:
    i, j, k = series.location
    lines = [f"# component={series.component} i={i} j={j} k={k} "
             f"bias_Apm={series.bias:.12e} dt_s={series.dt_sample:.12e}\n"]
    lines += [_FMT % v + "\n" for v in series.samples]
    path.write_text("".join(lines))


def cmd_simulate(args) -> int:
    started = time.time()
    config = load_config(args.config)
    if args.dry_run:
        fs, cs = config.grid.field_shape, config.grid.cell_shape
        print(f"dt = {config.dt:.6e} s")
        print(f"steps = {config.n_steps}")
        print(f"cells = {cs} ({np.prod(cs)} total)")
        print(f"field memory ~ {8 * (6 * np.prod(fs) + 3 * np.prod(cs)) / 1e6:.1f} MB")
        print(f"probes = {len(config.probes)}")
        return EXIT_OK
    out = _out_dir(args)
    result = sim.run(config)
    files = []
    for (comp, (i, j, k)), series in result.probes.items():
        p = out / f"probe_{comp}_{i}_{j}_{k}.txt"
        write_probe(p, series)
        files.append(p)
    its = result.iterations
    diag = {"steps": result.steps,
            "llg_iterations_median": float(np.median(its)) if its.size else None,
            "llg_iterations_max": int(its.max()) if its.size else None}
    _manifest(out, "simulate", args.config, files, started, diag)
    print(f"wrote {len(files)} probe files to {out}")
    return EXIT_OK


def cmd_sweep(args) -> int:
    started = time.time()
    config = load_config(args.config)
    biases = None
    if args.bias_start is not None:
        lo, hi = parse_quantity(args.bias_start), parse_quantity(args.bias_stop)
        step = parse_quantity(args.bias_step)
        count = int(math.floor((hi - lo) / step + 1e-9)) + 1
        biases = [lo + i * step for i in range(count)]
    if args.dry_run:
        n = len(biases if biases is not None else config.bias_sweep)
        print(f"sweep of {n} runs, {config.n_steps} steps each, dt = {config.dt:.6e} s")
        return EXIT_OK
    out = _out_dir(args)
    smap = sim.sweep(config, biases=biases, parallel=args.parallel)
    path = out / "spectrum_map.txt"
    rows = ["# bias_Apm frequency_Hz magnitude\n"]
    for bi, b in enumerate(smap.biases):
        rows += [f"{b:.12e} {fr:.12e} {mg:.12e}\n" for fr, mg in zip(smap.freqs, smap.mags[bi])]
    path.write_text("".join(rows))
    _manifest(out, "sweep", args.config, [path], started,
              {"n_bias": len(smap.biases), "n_freq": len(smap.freqs)})
    print(f"wrote {path}")
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="magphon-b200",
                                description="B200 coupled Maxwell-LLG stepper")
    p.add_argument("--seed", type=int, default=0, help="accepted for compatibility")
    p.add_argument("--parallel", type=int, default=1, help="concurrent sweep runs (spread over the GPUs, several per GPU)")
    p.add_argument("--dry-run", action="store_true")
    p.add_argument("--out", default=None, help="output directory ($MAGPHON_OUT or .)")
    sub = p.add_subparsers(dest="command", required=True)
    s = sub.add_parser("simulate", help="run one simulation from a config")
    s.add_argument("config")
    s.set_defaults(func=cmd_simulate)
    s = sub.add_parser("sweep", help="bias sweep -> spectrum map")
    s.add_argument("config")
    s.add_argument("--bias-start")
    s.add_argument("--bias-stop")
    s.add_argument("--bias-step")
    s.set_defaults(func=cmd_sweep)
    return p


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return EXIT_USAGE if exc.code not in (0, None) else EXIT_OK
    try:
        return args.func(args)
    except (ConfigError, ValueError, KeyError, IndexError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_USAGE
    except (StepFailure, FloatingPointError, RuntimeError) as exc:
        print(f"runtime failure: {exc}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
