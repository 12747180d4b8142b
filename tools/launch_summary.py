"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum
--csv --log-file): launches, total device time and share of the total. ncu
serializes launches and runs them cold-cache, so shares (not absolute times)
are what compares with bench.py's CUDA-event profile."""
import csv
import re
import sys
from collections import defaultdict

path = sys.argv[1]
rows = []
with open(path) as f:
    lines = [ln for ln in f if ln.startswith('"')]
rd = csv.reader(lines)
hdr = next(rd)
ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rd:
    if r[im] != "gpu__time_duration.sum":
        continue
    v = float(r[iv].replace(",", ""))
    unit = r[iu]
    ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v if unit in ("ms", "msecond") else v / 1e6
    name = re.sub(r"\(.*", "", r[ik])
    name = re.sub(r"^void ", "", name)
    tot[name] += ms
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"# {sum(cnt.values())} launches, {all_ms:.1f} ms device time (ncu: serialized, cold cache)")
print(f"{'kernel':70s} {'launches':>8s} {'ms':>11s} {'share':>7s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k[:70]:70s} {cnt[k]:8d} {tot[k]:11.2f} {100 * tot[k] / all_ms:6.2f}%")
