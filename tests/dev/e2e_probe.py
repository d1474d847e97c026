"""Dev: where does the e2e (pinned host input) step lose time vs the device-input step?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_1404_5997_b200 as hp

spec = hp.alexnet_1col()
c = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=128, seed=1, math_mode=hp.MathMode.BF16))
hyper = hp.HyperParams(momentum=0.9, lr=1e-4, weight_decay=5e-4)
NB = 4
host = [hp.synthetic_batch(spec, 128, step=s) for s in range(NB)]
dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()) for x, t in host]
pinned = [(torch.from_numpy(x).pin_memory(), torch.from_numpy(t).pin_memory()) for x, t in host]
stream = torch.cuda.ExternalStream(c.stream_ptr())
for kind in (dev, pinned):
    for s in range(2 * NB):
        x, t = kind[s % NB]
        if kind is pinned:
            c.prefetch([x], [t])
        c.run_step([x], [t], hyper, device=kind is dev)
torch.cuda.synchronize()


def loop(mode, steps=30):
    tp = tr = 0.0
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    if mode in ("host", "pref_dev"):
        c.prefetch([pinned[0][0]], [pinned[0][1]])
    e0.record(stream)
    for s in range(steps):
        a = time.perf_counter()
        if mode in ("host", "pref_dev") and s + 1 < steps:
            xn, tn = pinned[(s + 1) % NB]
            c.prefetch([xn], [tn])
        b = time.perf_counter()
        if mode == "host":
            x, t = pinned[s % NB]
            c.run_step([x], [t], hyper, device=False)
        else:
            x, t = dev[s % NB]
            c.run_step([x], [t], hyper, device=True)
        tp += b - a
        tr += time.perf_counter() - b
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    dev_ms = c.last_step_ms()
    print(f"{mode:9s}: {ms:.3f} ms/step (last step device {dev_ms:.3f}); host prefetch {tp / steps * 1e3:.3f} ms, "
          f"run_step call {tr / steps * 1e3:.3f} ms", flush=True)


for mode in ("device", "host", "pref_dev", "device", "host"):
    loop(mode)
