"""Developer: per-kernel table of one FGMRES iteration from an ncu launch list (--csv --log-file)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; data = rows[hi + 1:]
ki, mi, vi, idi = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
L = collections.OrderedDict()
for r in data:
    d = L.setdefault(r[idi], {'k': r[ki]})
    d[r[mi]] = float(r[vi].replace(',', ''))
launches = list(L.values())
names = [l['k'].split('(')[0] for l in launches]
idx = [i for i, n in enumerate(names) if 'k_dcgs_update' in n]
a, b = idx[-2] + 1, idx[-1] + 1
tot = sum(l['gpu__time_duration.sum'] for l in launches[a:b])
for l in launches[a:b]:
    t = l['gpu__time_duration.sum']
    print(f"{l['k'][:58]:58s} {t/1e3:8.1f} us {100*t/tot:5.1f}% {l.get('dram__bytes_read.sum',0)/1e6:9.1f} MB  grid {int(l.get('launch__grid_size',0))}")
print('launches', b - a, 'total', tot / 1e6, 'ms')
