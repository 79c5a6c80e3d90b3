"""Per-kernel counts of the Blackwell-native SASS instructions in
libdapple.so (cuobjdump -sass): tcgen05 MMAs (UTC*MMA), TMEM loads (LDTM),
TMA loads / stores / reduce-adds (UTMALDG / UTMASTG / UTMAREDG), bulk copies
(UBLKCP), legacy HMMA (should be 0).  python tools/sass_summary.py [lib]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2007_01045_b200", "libdapple.so")
text = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAREDG", "UBLKCP", "HMMA", "MUFU.EX2", "MUFU.TANH"]
kernels = collections.OrderedDict()
cur = None
for line in text.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        kernels[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    ins = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", line)
    if not ins:
        continue
    op = ins.group(1)
    for k in KEYS:
        if op == k or op.startswith(k + "."):
            kernels[cur][k] += 1


def short(name):
    d = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
    d = d.replace("(anonymous namespace)::", "").replace("dpl::", "")
    d = re.sub(r"^void ", "", d)
    d = re.sub(r"\(.*", "", d)
    return d


print(f"{'kernel':60s} " + " ".join(f"{k:>9s}" for k in KEYS))
for name, c in kernels.items():
    if not any(c.values()):
        continue
    print(f"{short(name)[:60]:60s} " + " ".join(f"{c[k]:9d}" for k in KEYS))
print(f"\n{len(kernels)} kernels in {os.path.basename(lib)}; rows shown: kernels with any counted instruction")
