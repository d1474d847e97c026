"""Predicted B200 (NVLink 5 / NVSwitch) weak-scaling table from cost_model,
compute calibrated to a measured 1-GPU AlexNet step. Usage:
  python tests/dev/cost_table.py [measured_step_ms_at_b128]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))

from paper_1404_5997_b200 import api as hp, cost_model as cm
from paper_1404_5997_b200.specs import alexnet_1col

ms = float(sys.argv[1]) if len(sys.argv) > 1 else 1.737
spec, p = alexnet_1col(), cm.b200_params()
scale = cm.calibrate(spec, 128, p, ms * 1e-3)
print(f"compute_scale={scale:.3f} (model FLOP time x scale = measured {ms} ms at b=128, K=1)")
print("| K | b | A | B | C | DP | best |")
print("|---|---|---|---|---|---|---|")
for K in (2, 4, 8):
    for b in (32, 64, 128, 256):
        row, best = [], None
        for s in (hp.Scheme.A, hp.Scheme.B, hp.Scheme.C, hp.Scheme.DP):
            r = cm.speedup(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=s), cm.b200_topology(K), p,
                           compute_scale=scale)
            row.append(r["speedup"] / K)
            if best is None or r["speedup"] > best[1]:
                best = (s.name, r["speedup"])
        print(f"| {K} | {b} | " + " | ".join(f"{e:.3f}" for e in row) + f" | {best[0]} |")
