"""Dev: summarise an HP_DEV_TIMELINE csv (one graph-replayed bench step): per
named kernel span begin/end relative to the step start, grouped by stream
(inferred from the name), and each stream's busy time."""
import collections, csv, sys

rows = list(csv.DictReader(open(sys.argv[1])))
step = int(sys.argv[2]) if len(sys.argv) > 2 else max(int(r["step"]) for r in rows)
rows = [r for r in rows if int(r["step"]) == step]
t0 = min(int(r["ns"]) for r in rows)
span = collections.OrderedDict()
for r in rows:
    t = (int(r["ns"]) - t0) / 1e3
    if r["kind"] == "point":
        span.setdefault(r["name"], [t, t])
        continue
    s = span.setdefault(r["name"], [None, None])
    s[0 if r["kind"] == "begin" else 1] = t
def stream(n):
    if n.startswith(("conv_wgrad", "colsum")): return "sw (conv wgrad)"
    if n.startswith("fc_wgrad"): return "sf (fc wgrad+sgd)"
    if n.startswith("marker"): return "markers"
    return "st (critical)"
by = collections.defaultdict(list)
for n, (a, b) in span.items():
    by[stream(n)].append((a if a is not None else b, b if b is not None else a, n))
end = max(b for v in by.values() for _, b, _ in v)
print(f"step {step}: {end:.1f} us from first to last marker")
for st, v in by.items():
    v.sort()
    busy = sum(b - a for a, b, _ in v)
    print(f"== {st}: busy {busy:.1f} us")
    for a, b, n in v:
        print(f"   {a:8.1f} {b:8.1f} {b - a:7.1f}  {n}")
