"""Dev: one-GPU step times of the K-worker schemes on the logical transport
(all K workers on one B200, collectives as device copies / ordered sums):
AlexNet-1col b=128 per worker, bf16, graphs. argv: K [schemes...]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1404_5997_b200 as hp

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cases = sys.argv[2:] or ["A", "B", "C", "Cv", "DP"]
spec = hp.alexnet_1col()
b = 128
xs, ts = zip(*[hp.synthetic_batch(spec, b, worker=w) for w in range(K)])
dx = [torch.from_numpy(x).cuda() for x in xs]
dt = [torch.from_numpy(t).cuda() for t in ts]
hyper = hp.HyperParams(momentum=0.9, lr=1e-4, weight_decay=5e-4)
for case in cases:
    scheme = {"A": hp.Scheme.A, "B": hp.Scheme.B, "C": hp.Scheme.C, "Cv": hp.Scheme.C, "DP": hp.Scheme.DP}[case]
    c = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=scheme, variable_batch=case == "Cv",
                                          seed=1, math_mode=hp.MathMode.BF16))
    for _ in range(4):
        c.run_step(dx, dt, hyper, device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    n = 10
    for _ in range(n):
        c.run_step(dx, dt, hyper, device=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"K={K} {case:3s} step {ms:7.3f} ms  ({K * b / ms * 1e3:8.0f} images/s on one B200)", flush=True)
    c.close()
    del c
