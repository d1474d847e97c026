"""Dev: per-kernel duration (us) and DRAM MB of the last of 3 eager steps in two
ncu --csv launch lists (gpu__time_duration.sum + dram bytes), side by side."""
import collections, csv, sys


def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-9, 'usecond': 1e-6,
                 'msecond': 1e-3, 'ns': 1e-9, 'us': 1e-6, 'ms': 1e-3}.get(r[ui], 1)
        per[int(r[ii])][r[mi]] = float(r[vi].replace(',', '')) * scale
        names[int(r[ii])] = r[ki].split('(')[0].replace('void ', '').replace('unnamed>::', '')[:58]
    ids = sorted(per)
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for i in ids[2 * len(ids) // 3:]:
        a = agg[names[i]]
        a[0] += per[i].get('gpu__time_duration.sum', 0) * 1e6
        a[1] += (per[i].get('dram__bytes_read.sum', 0) + per[i].get('dram__bytes_write.sum', 0)) / 1e6
    return agg


a, b = load(sys.argv[1]), load(sys.argv[2])
print(f"{'kernel':58s} {'old us':>8s} {'new us':>8s} {'oldMB':>7s} {'newMB':>7s}")
for k in sorted(set(a) | set(b), key=lambda k: -max(a.get(k, [0])[0], b.get(k, [0])[0])):
    x, y = a.get(k, [0, 0]), b.get(k, [0, 0])
    print(f"{k:58s} {x[0]:8.1f} {y[0]:8.1f} {x[1]:7.1f} {y[1]:7.1f}")
print(f"{'total':58s} {sum(v[0] for v in a.values()):8.1f} {sum(v[0] for v in b.values()):8.1f}")
