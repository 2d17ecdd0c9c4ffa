"""Per-kernel mean duration and DRAM bytes from an ncu --csv launch list.

    python tools/launch_table.py gpurun_out/launches_c3.csv
"""
import collections
import csv
import io
import sys

text = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
per = collections.defaultdict(lambda: collections.defaultdict(list))
for r in csv.DictReader(io.StringIO("\n".join(text[start:]))):
    per[r["Kernel Name"].split("(")[0]][r["Metric Name"]].append(
        float(r["Metric Value"].replace(",", "")))
total = sum(sum(d["gpu__time_duration.sum"]) for d in per.values())
print("| kernel | launches | mean ns | share | DRAM read B | DRAM write B |")
print("|---|---|---|---|---|---|")
for k, d in sorted(per.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    t = d["gpu__time_duration.sum"]
    n = len(t)
    print(f"| {k} | {n} | {sum(t)/n:.0f} | {100*sum(t)/total:.1f}% | "
          f"{sum(d['dram__bytes_read.sum'])/n:.3e} | {sum(d['dram__bytes_write.sum'])/n:.3e} |")
