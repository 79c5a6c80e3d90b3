"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv)."""
import collections
import csv
import re
import sys


def main(path, limit=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    n = 0
    for r in rows[1:]:
        if r[im] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ik]).split("::")[-1]
        name = re.sub(r"<.*", "", name)
        tot[name] += float(r[iv].replace(",", "")) / 1000.0
        cnt[name] += 1
        n += 1
    s = sum(tot.values())
    print(f"{n} launches profiled (ncu --metrics gpu__time_duration.sum, cold-cache serialised); share of profiled time:")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"  {k:36s} {cnt[k]:5d} launches {v:11.1f} us {100 * v / s:6.1f}%  avg {v / cnt[k]:8.2f} us")


if __name__ == "__main__":
    main(sys.argv[1])
