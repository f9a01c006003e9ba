"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import csv, collections, sys
path = sys.argv[1]
iters = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = list(csv.DictReader(l for l in open(path) if not l.startswith('==')))
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
for r in rows:
    if r.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    name = r['Kernel Name'].split('(')[0].replace('void ', '')
    agg[name][0] += 1
    agg[name][1] += float(r['Metric Value']) * scale[r['Metric Unit']]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'us/iter':>10s} {'avg us':>8s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:48]:48s} {n/iters:8.1f} {t/iters:10.1f} {t/n:8.2f} {100*t/tot:5.1f}%")
print(f"total {tot/iters:.1f} us per iteration (serialised, cold-cache ncu launches)")
