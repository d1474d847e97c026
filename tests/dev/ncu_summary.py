"""Summarise an ncu --set full report (raw page CSV) per launch: duration,
tensor-pipe activity, DRAM bytes, L2 (lts) throughput, TMA bytes."""
import csv, subprocess, sys

rep = sys.argv[1]
names = sys.argv[2].split(",") if len(sys.argv) > 2 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
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


def unit(k):
    return rows[1][col[k]] if k in col else ""


def scale(k, to):
    u = unit(k)
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9, "msecond": 1e-3,
         "usecond": 1e-6, "nsecond": 1e-9}.get(u, 1)
    return f / to


print(f"{'#':>3} {'kernel':34s} {'grid':>10s} {'us':>8s} {'tensor%':>7s} {'dramMB':>8s} {'dramTB/s':>8s} {'lts%':>5s} {'sm%':>5s} {'tmaGB':>7s}")
for n, r in enumerate(rows[2:]):
    name = r[col["Kernel Name"]]
    short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")[-34:]
    t = g(r, "gpu__time_duration.sum") * scale("gpu__time_duration.sum", 1e-6)
    rd = g(r, "dram__bytes_read.sum") * scale("dram__bytes_read.sum", 1e6)
    wr = g(r, "dram__bytes_write.sum") * scale("dram__bytes_write.sum", 1e6)
    ten = g(r, "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")
    if ten != ten:
        ten = g(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed")
    lts = g(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed")
    sm = g(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed")
    tma = g(r, "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum") * scale(
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", 1e9)
    grid = r[col["Grid Size"]] if "Grid Size" in col else ""
    print(f"{n:3d} {short:34s} {grid:>10s} {t:8.1f} {ten:7.1f} {rd + wr:8.1f} {(rd + wr) / t:8.2f} {lts:5.1f} {sm:5.1f} {tma:7.3f}")
