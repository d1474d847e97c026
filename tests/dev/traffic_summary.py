"""ncu per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum)
of the LAST eager step (tests/dev/one_step.py 2) -> profiles JSON: bytes per
step for the tcgen05 GEMM launches (bench.py's roofline 'traffic') and per kernel."""
import csv, collections, json, sys
src, out = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, mi, vi, ui, ii = (h.index(k) for k in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
per = collections.defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    scale = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'nsecond': 1e-9, 'usecond': 1e-6, 'msecond': 1e-3,
             'ns': 1e-9, 'us': 1e-6, 'ms': 1e-3}.get(r[ui], 1)
    per[int(r[ii])][r[mi]] = float(r[vi].replace(',', '')) * scale
    names[int(r[ii])] = r[ki].split('(')[0].replace('void ', '').replace('unnamed>::', '')
ids = sorted(per)
n = len(ids) // 2
last = ids[n:]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i in last:
    k = names[i]
    a = agg[k]
    a[0] += 1
    a[1] += per[i].get('dram__bytes_read.sum', 0) + per[i].get('dram__bytes_write.sum', 0)
    a[2] += per[i].get('gpu__time_duration.sum', 0)
gemm = sum(v[1] for k, v in agg.items() if 'gemm' in k or 'conv_shift' in k)
res = {"source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                  "python tests/dev/one_step.py 2 (last eager step, AlexNet-1col b=128 bf16, K=1)",
       "gemm_dram_bytes_per_step": gemm,
       "per_kernel": {k: {"launches": v[0], "dram_bytes": v[1], "us": v[2] * 1e6} for k, v in
                      sorted(agg.items(), key=lambda kv: -kv[1][2])}}
json.dump(res, open(out, 'w'), indent=1)
print(f"GEMM DRAM bytes/step {gemm / 1e6:.1f} MB")
for k, v in list(res["per_kernel"].items())[:12]:
    print(f"  {v['us']:8.1f} us {v['dram_bytes'] / 1e6:8.1f} MB {v['launches']:3d}  {k}")
