"""Developer: aggregate the setup-phase kernels of an ncu launch list (launches before the first FGMRES norm)."""
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
names = [l['k'].split('(')[0].replace('void ', '').replace('tsp::', '') for l in launches]
end = next(i for i, n in enumerate(names) if n.startswith('k_mdot') or n.startswith('k_op_node'))
agg = collections.defaultdict(lambda: [0, 0.0])
for n, l in zip(names[:end], launches[:end]):
    agg[n][0] += 1; agg[n][1] += l['gpu__time_duration.sum']
tot = sum(v[1] for v in agg.values())
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
    print(f"{n:40s} {c:6d} {t/1e6:9.2f} ms {100*t/tot:5.1f}%")
print('setup launches', end, 'kernel time', tot / 1e6, 'ms')
