"""Dev: step time and per-GEMM times with the GEMM epilogue's global traffic skipped
(dbg bit 0; results are garbage) -- how much of each GEMM is epilogue-bound."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1404_5997_b200 as hp
from paper_1404_5997_b200._lib import lib

spec = hp.alexnet_1col()
dev = [tuple(torch.from_numpy(a).cuda() for a in hp.synthetic_batch(spec, 128, step=s)) for s in range(4)]
hyper = hp.HyperParams(momentum=0.9, lr=1e-4, weight_decay=5e-4)
res = {}
FL = [int(a) for a in sys.argv[1:]] or [0, 1]
for flags in FL:
    lib.hp_debug_gemm_flags(flags)
    c = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=128, seed=1, math_mode=hp.MathMode.BF16))
    for s in range(10):
        c.run_step([dev[s % 4][0]], [dev[s % 4][1]], hyper, device=True)
    ms = []
    for s in range(20):
        c.run_step([dev[s % 4][0]], [dev[s % 4][1]], hyper, device=True)
        ms.append(c.last_step_ms())
    c.set_profile(True)
    per = {}
    for s in range(3):
        c.run_step([dev[s % 4][0]], [dev[s % 4][1]], hyper, device=True)
        for tag, layer, flops, pms in c.gemm_profile():
            per[f"{tag}[{layer}]"] = per.get(f"{tag}[{layer}]", 0.0) + pms / 3
    res[flags] = (np.median(ms), per)
    c.close()
lib.hp_debug_gemm_flags(0)
print("step ms per dbg flags:", {f: round(res[f][0], 4) for f in FL})
for k in sorted(res[FL[0]][1], key=lambda k: -res[FL[0]][1][k]):
    print(f"  {k:16s} " + " ".join(f"{res[f][1].get(k, 0) * 1e3:7.1f}" for f in FL))
