"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel count, time, share."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[hi]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = re.sub(r"\(.*", "", r[ki])
    name = re.sub(r"rk::<unnamed>::|void |at::", "", name)
    v = float(r[vi].replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3,
                                            "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1.0)
    tot[name] += v
    cnt[name] += 1
T = sum(tot.values())
print(f"{sum(cnt.values())} launches, {T / 1e3:.1f} ms of kernel time (cold-cache, serialised)")
print(f"{'kernel':58s} {'launches':>8s} {'ms':>10s} {'share':>6s} {'avg us':>9s}")
for k, v in tot.most_common():
    print(f"{k[:58]:58s} {cnt[k]:8d} {v / 1e3:10.2f} {100 * v / T:5.1f}% {v / cnt[k]:9.1f}")
