"""Dev harness for ncu: N eager (no CUDA graph) AlexNet-1col bf16 steps, b=128,
K=1, scheme B exact -- the bench workload, launch order deterministic."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1404_5997_b200 as hp

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
spec = hp.alexnet_1col()
c = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=128, scheme=hp.Scheme.B, seed=1,
                                      math_mode=hp.MathMode.BF16))
c.set_graphs(False)
x, t = hp.synthetic_batch(spec, 128)
x, t = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
hyper = hp.HyperParams(momentum=0.9, lr=0.0001, weight_decay=5e-4)
for s in range(steps):
    r = c.run_step([x], [t], hyper, device=True)
torch.cuda.synchronize()
print("loss", r.metrics.loss, "launches/step", c.last_step_launches())
