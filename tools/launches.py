"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
gi = hdr.index('Grid Size') if 'Grid Size' in hdr else None
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].replace('void ', '')[:48]
    if gi is not None:
        name += ' ' + r[gi]
    v = float(r[vi].replace(',', ''))
    v = v / 1000 if r[ui] == 'ns' else (v * 1000 if r[ui] in ('ms', 'msecond') else v)
    agg[name].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:75s} n={len(v):4d} mean={sum(v)/len(v):9.1f}us total={sum(v):10.1f}us {100*sum(v)/tot:5.1f}%")
