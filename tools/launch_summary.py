"""Aggregate an ncu `--metrics gpu__time_duration.sum --csv` launch list per kernel."""
import collections, csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
agg, seq = collections.OrderedDict(), []
for row in csv.DictReader(lines):
    k = row['Kernel Name'].split('(')[0]
    v = float(row['Metric Value'].replace(',', ''))
    u = row['Metric Unit']
    ms = v / 1e6 if u.startswith('ns') else (v / 1e3 if u.startswith('us') else v)
    agg.setdefault(k, [0, 0.0]); agg[k][0] += 1; agg[k][1] += ms
    seq.append((k, ms))
tot = sum(v[1] for v in agg.values())
for k, v in agg.items():
    print(f"{k:40s} n={v[0]:4d} total={v[1]:9.3f} ms  {100*v[1]/tot:5.1f}%")
print(f"total {tot:.3f} ms")
if len(sys.argv) > 2:
    for name in sys.argv[2:]:
        print(name, [round(ms, 2) for k, ms in seq if k == name])
