"""Dev (GPU): cost-model phase split vs the measured 1-GPU step. Measured:
per-GEMM CUDA-event times (library profile pass) summed by phase, plus the
whole step; model: cost_model's K=1 timeline calibrated to the measured step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1404_5997_b200 as hp
from paper_1404_5997_b200 import cost_model as cm

spec = hp.alexnet_1col()
c = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=128, seed=1, math_mode=hp.MathMode.BF16))
dev = [tuple(torch.from_numpy(a).cuda() for a in hp.synthetic_batch(spec, 128, step=s)) for s in range(4)]
hyper = hp.HyperParams(momentum=0.9, lr=1e-4, weight_decay=5e-4)
for s in range(10):
    c.run_step([dev[s % 4][0]], [dev[s % 4][1]], hyper, device=True)
ms = []
for s in range(20):
    c.run_step([dev[s % 4][0]], [dev[s % 4][1]], hyper, device=True)
    ms.append(c.last_step_ms())
step = float(np.median(ms))
c.set_profile(True)
ph = {"conv_fwd": 0.0, "fc": 0.0, "conv_bwd": 0.0}
for s in range(3):
    c.run_step([dev[s % 4][0]], [dev[s % 4][1]], hyper, device=True)
    for tag, layer, flops, pms in c.gemm_profile():
        key = "conv_fwd" if tag == "conv_fwd" else ("fc" if tag.startswith("fc") else "conv_bwd")
        ph[key] += pms / 3
p = cm.b200_params()
scale = cm.calibrate(spec, 128, p, step * 1e-3)
tl = cm.scheme_step_model(spec, hp.ClusterConfig(workers=1, per_worker_batch=128), cm.Topology(1), p, scale)
model = tl.phase_table()
model["fc"] = model.get("fc", 0.0) + model.get("fc_update", 0.0)  # the measured FC GEMMs include the fused update
tot_g = sum(ph.values())
print(f"measured step {step:.3f} ms; GEMM time {tot_g:.3f} ms; calibration scale {scale:.3f}")
print(f"{'phase':10s} {'model ms':>9s} {'model %':>8s} {'GEMM ms':>8s} {'GEMM %':>7s}")
for k in ("conv_fwd", "fc", "conv_bwd"):
    print(f"{k:10s} {model[k] * 1e3:9.3f} {model[k] / tl.step_time * 100:7.1f}% {ph[k]:8.3f} {ph[k] / tot_g * 100:6.1f}%")
