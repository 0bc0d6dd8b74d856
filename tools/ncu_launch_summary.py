"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list per kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
scale = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    except ValueError:
        continue
    nm = r[ki].split('(')[0]
    agg[nm][0] += 1
    agg[nm][1] += v
tot = sum(t for _, t in agg.values())
title = sys.argv[2] if len(sys.argv) > 2 else ''
print(f"# {title}\n# per-kernel totals from ncu launch list (cold-cache, serialised: compare SHARES)")
print(f"{'kernel':48s} {'launches':>8s} {'total_us':>10s} {'us/launch':>10s} {'share':>7s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:48]:48s} {n:8d} {t:10.1f} {t / n:10.2f} {100 * t / tot:6.1f}%")
