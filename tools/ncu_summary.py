"""Summarise ncu outputs from gpurun_out/ into profiles/ (committed evidence).

    python tools/ncu_summary.py r01

Writes profiles/<tag>_launches.csv (per-launch durations + DRAM bytes of the
bench command), profiles/<tag>_sweep_summary.md (headline metrics of the full
k_sweep capture) and updates profiles/traffic.json (DRAM bytes per launch of
the dominant kernel, read by bench.py as roofline.traffic).
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"


def launches(tag):
    src = OUT / f"launches_{tag}.csv"
    text = src.read_text().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    per = defaultdict(dict)
    for r in rows:
        per[(int(r["ID"]), r["Kernel Name"].split("(")[0])][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    lines = ["id,kernel,duration_ns,dram_read_bytes,dram_write_bytes"]
    agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for (i, k), m in sorted(per.items()):
        d = m.get("gpu__time_duration.sum", 0.0)
        rb = m.get("dram__bytes_read.sum", 0.0)
        wb = m.get("dram__bytes_write.sum", 0.0)
        lines.append(f"{i},{k},{d:.0f},{rb:.0f},{wb:.0f}")
        a = agg[k]
        a[0] += 1; a[1] += d; a[2] += rb; a[3] += wb
    (PROF / f"{tag}_launches.csv").write_text("\n".join(lines) + "\n")
    tot = sum(a[1] for a in agg.values())
    share = {k: {"launches": a[0], "total_ns": a[1], "share": a[1] / tot,
                 "dram_bytes_per_launch": (a[2] + a[3]) / a[0]} for k, a in agg.items()}
    return share


_SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
          "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def raw_metrics(rep):
    """name -> (value, unit) from the raw page; bytes/seconds normalised."""
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    res = {}
    for name, unit, val in zip(h, u, v):
        try:
            x = float(val.replace(",", ""))
        except ValueError:
            res[name] = (val, unit)
            continue
        if unit in _SCALE:
            x *= _SCALE[unit]
            unit = "byte" if "byte" in unit else "second"
        res[name] = (x, unit)
    return res


def main(tag, dtype="f64"):
    PROF.mkdir(exist_ok=True)
    share = launches(tag)
    rep = OUT / f"sweep_{tag}.ncu-rep"
    m = raw_metrics(rep)
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__average_warp_latency_issue_stalled_barrier",
            "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]
    lines = [f"# ncu summary -- k_sweep ({tag})", "",
             f"Command: `python bench.py --steps 6 --warmup 3 --no-cpu"
             f"{' --dtype f32' if dtype == 'f32' else ''}` (C4 1024x1024x128, "
             f"{'fp64' if dtype == 'f64' else 'fp32 E/H storage'}),",
             "kernel launch #4 (after warm-up), `ncu --set full --clock-control none`.", "",
             "| metric | value |", "|---|---|"]
    for k in keys:
        if k in m:
            val, unit = m[k]
            txt = f"{val:.6g}" if isinstance(val, float) else val
            lines.append(f"| `{k}` | {txt} {unit} |")
    lines += ["", "## Launch list share (same command, cold-cache serialised)", "",
              "| kernel | launches | share of GPU time | DRAM bytes / launch |", "|---|---|---|---|"]
    for k, a in sorted(share.items(), key=lambda kv: -kv[1]["share"]):
        lines.append(f"| {k} | {a['launches']} | {100 * a['share']:.1f}% | {a['dram_bytes_per_launch']:.3e} |")
    (PROF / f"{tag}_sweep_summary.md").write_text("\n".join(lines) + "\n")
    traffic = {}
    tp = PROF / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text())
    rb = m["dram__bytes_read.sum"][0]
    wb = m["dram__bytes_write.sum"][0]
    traffic["k_sweep" if dtype == "f64" else f"k_sweep_{dtype}"] = rb + wb
    traffic[f"_source_{dtype}"] = f"profiles/{tag}_sweep_summary.md (ncu --set full, one launch)"
    tp.write_text(json.dumps(traffic, indent=1) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", sys.argv[2] if len(sys.argv) > 2 else "f64")
