"""Dev harness (GPU): AlexNet-1col step timing with per-GEMM split, fused vs
unfused FC SGD, and loss trajectories per learning rate / math mode."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1404_5997_b200 as hp

spec = hp.alexnet_1col()
what = sys.argv[1] if len(sys.argv) > 1 else "time"


def make(math=hp.MathMode.BF16, b=128, scheme="B"):
    cfg = hp.ClusterConfig(workers=1, per_worker_batch=b, scheme=hp.Scheme.from_string(scheme), seed=1, math_mode=math)
    return hp.Cluster(spec, cfg)


batches = [hp.synthetic_batch(spec, 128, step=s) for s in range(4)]
dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()) for x, t in batches]

if what == "time":
    for fuse, shift in ((True, True), (True, False)):
        c = make()
        c.set_fuse_fc_sgd(fuse)
        c.set_shift_conv(shift)
        hyper = hp.HyperParams(momentum=0.9, lr=0.001, weight_decay=5e-4)
        for s in range(12):
            x, t = dev[s % 4]
            c.run_step([x], [t], hyper, device=True)
        torch.cuda.synchronize()
        ms = []
        for s in range(20):
            x, t = dev[s % 4]
            c.run_step([x], [t], hyper, device=True)
            ms.append(c.last_step_ms())
        c.set_profile(True)
        per = {}
        for s in range(3):
            x, t = dev[s % 4]
            c.run_step([x], [t], hyper, device=True)
            for tag, layer, flops, pms in c.gemm_profile():
                a = per.setdefault(f"{tag}[{layer}]", [0.0, 0.0])
                a[0] += flops / 3
                a[1] += pms / 3
        c.set_profile(False)
        tot = sum(v[1] for v in per.values())
        print(f"fuse={fuse} shift={shift}: step {np.median(ms):.3f} ms (min {min(ms):.3f}), gemm {tot:.3f} ms, "
              f"{128 / np.median(ms) * 1e3:.0f} img/s")
        for k, (f, t) in sorted(per.items(), key=lambda kv: -kv[1][1]):
            print(f"   {k:16s} {t:7.3f} ms {f / 1e9:7.2f} GF {f / t / 1e9:7.1f} TF/s")
        c.close()
elif what == "loss":
    for math in (hp.MathMode.BF16, hp.MathMode.F32X3):
        for lr in (0.001, 0.0003, 0.0001):
            c = make(math)
            hyper = hp.HyperParams(momentum=0.9, lr=lr, weight_decay=5e-4)
            ls = []
            for s in range(90):
                x, t = dev[s % 4]
                r = c.run_step([x], [t], hyper, device=True)
                ls.append(r.metrics.loss)
            print(f"math={math} lr={lr}: " + " ".join(f"{v:.4g}" for v in ls[::3]), flush=True)
            c.close()
