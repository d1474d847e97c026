"""Summarise an ncu --set full capture per launch (raw page CSV: a .ncu-rep, or the
exported .csv / .csv.gz): duration, tcgen05 tensor activity, DRAM bytes, L2->SM
bytes, L2 throughput.

tensor% is the bf16->fp32 tensor-op path utilisation
(sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off, % of peak over the
elapsed time) -- the counter tcgen05.mma kind::f16 drives on sm_100. memT% is
sm__mem_tensor_cycles_active (tensor-core operand reads from smem/TMEM). The
legacy sm__pipe_tensor_cycles_active counts only the HMMA (mma.sync) pipe and
reads ~3% on tcgen05 kernels, so it is not used.
usage: ncu_summary.py <rep|csv|csv.gz> [labels comma-separated | --mem]
--mem: the memory-kernel table (us, DRAM MB and TB/s, issue%, achieved occupancy, sm% / l1%)."""
import csv, gzip, io, subprocess, sys

src = sys.argv[1]
mem = len(sys.argv) > 2 and sys.argv[2] == "--mem"
labels = sys.argv[2].split(",") if len(sys.argv) > 2 and not mem else None
if src.endswith(".ncu-rep"):
    text = subprocess.run(["ncu", "-i", src, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
elif src.endswith(".gz"):
    text = gzip.open(src, "rt").read()
else:
    text = open(src).read()
rows = list(csv.reader(io.StringIO(text)))
h = rows[0]
col = {k: i for i, k in enumerate(h)}


def g(r, k, default=float("nan")):
    i = col.get(k)
    if i is None or i >= len(r) or r[i] in ("", "n/a"):
        return default
    try:
        return float(r[i].replace(",", ""))
    except ValueError:
        return default


def scale(k, to):
    u = rows[1][col[k]] if k in col else ""
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "msecond": 1e-3,
         "usecond": 1e-6, "nsecond": 1e-9}.get(u, 1)
    return f / to


if mem:
    print(f"{'kernel':50s} {'us':>6s} {'dramMB':>7s} {'TB/s':>5s} {'issue%':>6s} {'warps%':>6s} {'sm%':>5s} {'l1%':>5s}")
    for r in rows[2:]:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("hp::", "")[-50:]
        t = g(r, "gpu__time_duration.sum") * scale("gpu__time_duration.sum", 1e-6)
        dram = (g(r, "dram__bytes_read.sum") * scale("dram__bytes_read.sum", 1e6) +
                g(r, "dram__bytes_write.sum") * scale("dram__bytes_write.sum", 1e6))
        print(f"{name:50s} {t:6.1f} {dram:7.1f} {dram / t:5.2f} {g(r, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):6.1f} "
              f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
              f"{g(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f} "
              f"{g(r, 'l1tex__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}")
    sys.exit(0)
TEN = "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed"
MEMT = "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
print(f"{'#':>3} {'label':12s} {'kernel':28s} {'grid':>6s} {'us':>7s} {'tensor%':>7s} {'memT%':>6s} {'dramMB':>7s} "
      f"{'TB/s':>5s} {'L2->SM MB':>9s} {'B/clk/SM':>8s} {'lts%':>5s}")
for n, r in enumerate(rows[2:]):
    name = r[col["Kernel Name"]]
    short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("hp::", "")[-28:]
    t = g(r, "gpu__time_duration.sum") * scale("gpu__time_duration.sum", 1e-6)
    dram = (g(r, "dram__bytes_read.sum") * scale("dram__bytes_read.sum", 1e6) +
            g(r, "dram__bytes_write.sum") * scale("dram__bytes_write.sum", 1e6))
    x2l1 = g(r, "l1tex__m_xbar2l1tex_read_bytes.sum") * scale("l1tex__m_xbar2l1tex_read_bytes.sum", 1e6)
    clk = g(r, "gpc__cycles_elapsed.max")
    sms = g(r, "device__attribute_multiprocessor_count", 148)
    bpc = x2l1 * 1e6 / (clk * sms) if clk == clk and clk > 0 else float("nan")
    grid = r[col["Grid Size"]].split(",")[0].strip("( ") if "Grid Size" in col else ""
    lab = labels[n] if labels and n < len(labels) else ""
    print(f"{n:3d} {lab:12s} {short:28s} {grid:>6s} {t:7.1f} {g(r, TEN):7.1f} {g(r, MEMT):6.1f} {dram:7.1f} "
          f"{dram / t:5.2f} {x2l1:9.1f} {bpc:8.1f} {g(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f}")
