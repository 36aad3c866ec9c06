"""Aggregate an ncu --metrics gpu__time_duration.sum launch list (CSV) by kernel."""
import csv, collections, sys
rows = [l for l in open(sys.argv[1]) if not l.startswith('==')]
agg = collections.defaultdict(lambda: [0, 0.0])
for x in csv.DictReader(rows):
    if x['Metric Name'] != 'gpu__time_duration.sum':
        continue
    v = float(x['Metric Value'].replace(',', ''))
    v *= {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'second': 1e6}.get(x['Metric Unit'], 1.0)
    nm = x['Kernel Name'].split('(')[0].replace('void ', '')[:48]
    agg[nm][0] += 1
    agg[nm][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'total_us':>12s} {'us/launch':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:48s} {v[0]:8d} {v[1]:12.1f} {v[1]/v[0]:10.1f} {v[1]/tot:6.3f}")
