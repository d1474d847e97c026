"""Dev: hash of every parameter after 3 bf16 AlexNet steps (compare kernel variants
bit-for-bit across processes, e.g. with / without HP_DEV_* switches)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1404_5997_b200 as hp

spec = hp.alexnet_1col()
c = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=128, seed=1, math_mode=hp.MathMode.BF16))
hyper = hp.HyperParams(momentum=0.9, lr=1e-3, weight_decay=5e-4)
for s in range(3):
    x, t = hp.synthetic_batch(spec, 128, step=s)
    r = c.run_step([x], [t], hyper)
h = hashlib.sha256()
for which in range(4):
    n = len(spec.conv_layers) if which < 2 else len(spec.fc_layers)
    for l in range(n):
        h.update(np.ascontiguousarray(c.param(0, which, l)).tobytes())
print(f"loss {r.metrics.loss:.9f} params sha256 {h.hexdigest()[:16]}")
