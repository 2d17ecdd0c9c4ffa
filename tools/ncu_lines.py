"""Per-source-line stall / instruction breakdown of an ncu capture.

    python tools/ncu_lines.py gpurun_out/sweep_r01d.ncu-rep [N]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 8
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr = None
idx = {}
cols = []
cur = None
fname = "?"
agg = collections.defaultdict(collections.Counter)
src = {}
for x in r:
    if not x:
        continue
    if x[0] == "File Path":
        fname = x[1].rsplit("/", 1)[-1]
        continue
    if x[0] == "Function Name":
        continue
    if x[0] == "Line No":
        hdr = x
        idx = {h: i for i, h in enumerate(hdr)}
        cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if x[0]:
        cur = f"{fname}:{x[0]}"
        src[cur] = x[1]
        continue
    if hdr is None or len(x) < len(hdr) or x[2] in ("...", ""):
        continue
    for c in cols + ["Instructions Executed"]:
        try:
            agg[cur][c] += int(x[idx[c]])
        except ValueError:
            pass
tot = collections.Counter()
for a in agg.values():
    tot.update(a)
allt = sum(tot[c] for c in cols)
print("stall mix:", {c[6:]: round(tot[c] / allt * 100, 1) for c in cols if tot[c]})
for c in ["stall_wait", "stall_long_sb", "stall_barrier", "stall_short_sb", "stall_selected",
          "stall_not_selected", "Instructions Executed"]:
    den = allt if c.startswith("stall") else tot[c]
    print("==", c)
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][c])[:top]:
        print(f"  {a[c] * 100 / den:5.1f}% {k:>20} {src[k].strip()[:80]}")
