"""Write a profiles/ summary: ncu launch-list shares per kernel (per step), the
bench JSON line and the per-GEMM event timings (bench --profile-out)."""
import csv, collections, json, sys
launches, bench_log, prof, out, title = sys.argv[1:6]
rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
data = [r for r in rows[hi + 1:] if len(r) > vi]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    name = r[ki].split('(')[0].replace('void ', '').replace('unnamed>::', '').replace('(anonymous namespace)::', '')
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(',', '')) / 1e3
tot = sum(v for c, v in agg.values())
steps = agg[[k for k in agg if 'xent' in k][0]][0]
lines = [f"# {title}", "# ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3",
         f"# {len(data)} launches over {steps} steps (graph priming + warmup + timed + e2e + profiled); cold-cache,",
         "# serialised per-launch times -> the SHARE of the step is what to read, not the absolute.",
         "  us/step  share  launches/step  kernel"]
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    lines.append(f"{v / steps:9.1f} {100 * v / tot:5.1f}% {c / steps:8.1f}      {k}")
lines.append(f"total {tot / steps:.1f} us/step (ncu, serialised)")
lines.append("")
lines.append("# bench.py --steps 20 --warmup 5 (same build, no profiler):")
lines += [l for l in open(bench_log) if l.startswith('{')]
p = json.load(open(prof))
lines.append("")
lines.append(f"# per-GEMM CUDA-event timing on the library stream (bench --profile-out): step {p['step_ms']:.3f} ms, "
             f"GEMMs {p['gemm_ms_per_step']:.3f} ms")
for k, v in sorted(p['per_gemm'].items(), key=lambda kv: -kv[1]['ms_per_step']):
    lines.append(f"{k:16s} {v['ms_per_step']:.3f} ms {v['gflop']:8.2f} GFLOP {v['tflops']:7.1f} TFLOP/s")
open(out, 'w').write("\n".join(lines) + "\n")
print("\n".join(lines[:12]))
