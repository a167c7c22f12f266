"""Developer: per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file).
usage: launch_summary.py launches.csv[.gz] [first_kernel_substring]
With a substring, only the launches from its first occurrence on are counted (e.g. skip the setup phase)."""
import collections, csv, gzip, sys
op = gzip.open if sys.argv[1].endswith(".gz") else open
with op(sys.argv[1], "rt") as f:
    rows = [r for r in csv.reader(l for l in f if l.startswith('"'))]
h, data = rows[0], rows[1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
start = 0
if len(sys.argv) > 2:
    start = next(i for i, r in enumerate(data) if sys.argv[2] in r[ki])
tot = collections.OrderedDict()
for r in data[start:]:
    nm = r[ki].split("(")[0].replace("void ", "").replace("tsp::", "")
    ns = float(r[vi].replace(",", "")) * {"ns": 1.0, "us": 1e3, "ms": 1e6}.get(r[ui], 1.0)
    t = tot.setdefault(nm, [0, 0.0])
    t[0] += 1; t[1] += ns
T = sum(v[1] for v in tot.values())
print(f"{len(data) - start} launches, {T / 1e6:.2f} ms of kernel time (cold-cache, serialised)")
print(f"{'kernel':44s} {'launches':>8s} {'ms':>10s} {'share':>7s} {'us/launch':>10s}")
for nm, (n, ns) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{nm[:44]:44s} {n:8d} {ns / 1e6:10.3f} {100 * ns / T:6.2f}% {ns / n / 1e3:10.1f}")
