import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1404_5997_b200 as hp
spec = hp.alexnet_1col()
for math, b, lr in [(hp.MathMode.BF16, 128, 0.01), (hp.MathMode.F32X3, 128, 0.01), (hp.MathMode.BF16, 128, 0.001), (hp.MathMode.BF16, 32, 0.01)]:
    g = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=b, seed=1, math_mode=math))
    hpar = hp.HyperParams(momentum=0.9, lr=lr, weight_decay=5e-4)
    losses = []
    for s in range(16):
        x, t = hp.synthetic_batch(spec, b, step=s % 4)
        r = g.run_step([x], [t], hpar)
        losses.append(r.metrics.loss)
        if not np.isfinite(r.metrics.loss):
            break
    mx = {f"c{l}": float(np.abs(g.param(0, 0, l)).max()) for l in range(5)}
    mx.update({f"f{l}": float(np.abs(g.param(0, 2, l)).max()) for l in range(3)})
    mx.update({f"fb{l}": float(np.abs(g.param(0, 3, l)).max()) for l in range(3)})
    print(math, b, lr, ["%.3f" % v for v in losses], mx, flush=True)
