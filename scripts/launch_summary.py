"""Per-kernel shares of one forward from an ncu launch list.

usage: launch_summary.py LAUNCHES.csv [forward_index]

LAUNCHES.csv is `ncu --metrics gpu__time_duration.sum --csv --log-file ...` of a
bench.py run. A forward starts at k4_patch_gather; forward_index picks which one
(default: the 4th = the timed step after 3 warm-ups). ncu times are cold-cache
and serialised: compare shares, not absolute times, with bench.py.
"""
import collections
import csv
import sys

rows = []
with open(sys.argv[1]) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        unit = r.get("Metric Unit", "")
        v = float(r["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}[unit]
        rows.append((r["Kernel Name"].split("(")[0], v * scale))
starts = [i for i, (n, _) in enumerate(rows) if n.startswith("k4_patch_gather") or "patch_gather" in n]
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if len(starts) <= k:
    sys.exit(f"only {len(starts)} forwards in the list")
a = starts[k]
b = starts[k + 1] if k + 1 < len(starts) else len(rows)
win = rows[a:b]
tot = sum(v for _, v in win)
agg = collections.defaultdict(lambda: [0, 0.0])
for n, v in win:
    agg[n][0] += 1
    agg[n][1] += v
print(f"forward #{k}: {len(win)} kernel launches, {tot / 1e3:.2f} ms (ncu, serialised, cold cache)")
print(f"{'kernel':60s} {'n':>4s} {'total ms':>9s} {'share':>6s} {'us/launch':>10s}")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n[:60]:60s} {c:4d} {v / 1e3:9.3f} {v / tot * 100:5.1f}% {v / c:10.1f}")
