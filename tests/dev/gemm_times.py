"""Dev: per-GEMM CUDA-event times of the bench step (AlexNet-1col b=128 bf16, K=1,
scheme B; profile mode serialises the side streams), mean over 3 steps, and the
plain step time with graphs. Env toggles (HP_DEV_*) select kernel variants."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_1404_5997_b200 as hp

if os.environ.get("HP_DEV_GEMM_DBG"):
    from paper_1404_5997_b200._lib import lib as _l
    _l.hp_debug_gemm_flags(int(os.environ["HP_DEV_GEMM_DBG"]))
spec = hp.alexnet_1col()
c = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=128, scheme=hp.Scheme.B, seed=1,
                                      math_mode=hp.MathMode.BF16))
x, t = hp.synthetic_batch(spec, 128)
x, t = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
hyper = hp.HyperParams(momentum=0.9, lr=0.0001, weight_decay=5e-4)
for _ in range(6):
    c.run_step([x], [t], hyper, device=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(20):
    c.run_step([x], [t], hyper, device=True)
e1.record(); torch.cuda.synchronize()
step = e0.elapsed_time(e1) / 20
c.set_profile(True)
acc = {}
for _ in range(3):
    c.run_step([x], [t], hyper, device=True)
    for tag, layer, flops, ms in c.gemm_profile():
        a = acc.setdefault(f"{tag}[{layer}]", [0.0, flops])
        a[0] += ms / 3
tot = sum(v[0] for v in acc.values())
label = os.environ.get("LABEL", "")
print(f"== {label} step {step:.4f} ms  gemm sum {tot:.4f} ms")
for k, (ms, fl) in acc.items():
    print(f"{label:10s} {k:16s} {ms * 1e3:7.1f} us {fl / ms / 1e9:7.0f} TF/s")
