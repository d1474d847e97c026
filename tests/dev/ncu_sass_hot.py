"""Top stall-sampled SASS lines of one kernel in an ncu report (source page)."""
import csv, subprocess, sys
rep, skip = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", skip, "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h) and r[0] != "Address"]
si = h.index("Warp Stall Sampling (All Samples)")
ex = h.index("Instructions Executed")
f = lambda x: float(x.replace(",", "")) if x not in ("", None) else 0.0
tot = sum(f(r[si]) for r in data)
print(rows[0][1][:120], "samples", tot)
for i, r in sorted(enumerate(data), key=lambda t: -f(t[1][si]))[:n]:
    print(f"{f(r[si]) / tot * 100:5.1f}% [{i:5d}] exec={r[ex]:>10s} {r[1][:100]}")
