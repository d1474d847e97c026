"""Per-kernel table of the LAST step in an ncu launch-list CSV (eager steps)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value'); gi = h.index('Grid Size')
data = [r for r in rows[hi + 1:] if len(r) > vi]
n = len(data) // steps
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in data[-n:]:
    v = float(r[vi].replace(',', '')) / 1e3
    tot += v
    name = r[ki].split('(')[0].replace('void ', '').replace('unnamed>::', '').replace('(anonymous namespace)::', '')
    agg[name][0] += 1
    agg[name][1] += v
for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{v:9.1f} us {100 * v / tot:5.1f}% {c:4d}  {k[:80]}")
print(f"total {tot:.1f} us over {n} launches")
