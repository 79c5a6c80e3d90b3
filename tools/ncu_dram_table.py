"""Per-kernel DRAM bytes / time / bandwidth from ncu --csv metric logs
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum,
dram__throughput.avg.pct_of_peak_sustained_elapsed).
    python tools/ncu_dram_table.py log.csv [log2.csv ...]"""
import collections
import csv
import re
import sys

per = collections.defaultdict(lambda: collections.defaultdict(list))
for path in sys.argv[1:]:
    hdr = None
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        k = re.sub(r"\(.*", "", d["Kernel Name"]).replace("unnamed>::", "").replace("dpl::", "").replace("void ", "")
        per[(k, d["Grid Size"])][d["Metric Name"]].append(float(d["Metric Value"].replace(",", "")))
print(f"{'kernel':36s} {'grid':>14s}  n  time_us  DRAM_MB  TB/s  dram%")
for (k, g), m in sorted(per.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
    n = len(m["gpu__time_duration.sum"])
    t = sum(m["gpu__time_duration.sum"]) / n / 1e3
    b = (sum(m["dram__bytes_read.sum"]) + sum(m["dram__bytes_write.sum"])) / n
    pct = sum(m["dram__throughput.avg.pct_of_peak_sustained_elapsed"]) / n
    print(f"{k[:36]:36s} {g:>14s} {n:2d} {t:8.2f} {b / 1e6:8.2f} {b / t / 1e6:5.2f} {pct:6.1f}")
