"""Dev: AlexNet bf16 step vs the bf16-storage oracle with the GPU's decisions replayed (prints)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
import paper_1404_5997_b200 as hp

spec = hp.alexnet_1col()
b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
lr = 0.01
print("cpus", os.cpu_count(), flush=True)
x, t = hp.synthetic_batch(spec, b, step=0, worker=0)
g = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=b, scheme=hp.Scheme.B, seed=1, math_mode=hp.MathMode.BF16))
r = g.run_step([x], [t], hp.HyperParams(momentum=0.9, lr=lr, weight_decay=5e-4))
o = O.OracleCluster(spec, workers=1, per_worker_batch=b, scheme="B", precision="single", seed=1)
o.set_storage_rounding("bf16")
forced = []
for l, c in enumerate(spec.conv_layers):
    o.force_decisions(0, 0, l, g.decisions(0, 0, l)); forced.append((0, l))
    if c.pool_kernel:
        o.force_decisions(0, 1, l, g.decisions(0, 1, l)); forced.append((1, l))
for l, f in enumerate(spec.fc_layers):
    if f.relu:
        o.force_decisions(0, 2, l, g.decisions(0, 2, l)); forced.append((2, l))
t0 = time.time()
m = o.run_step([x.astype(np.float64)], [t.astype(np.float64)], O.make_hyper_c(0.9, lr, 5e-4))
print(f"oracle step {time.time() - t0:.1f} s; loss {r.metrics.loss:.10f} / {m.loss:.10f}")
for kind, l in forced:
    mis, gap = o.decision_stats(0, kind, l)
    n = g.decisions(0, kind, l).size
    print(f"  decisions kind {kind} layer {l}: {mis}/{n} differ ({mis / n:.2e}), max gap {gap:.2e}")
for which in (4, 5, 6, 7):
    for l in range(5 if which < 6 else 3):
        v = g.param(0, which, l).astype(np.float64)
        rv = o.param(0, which, l)
        e = np.abs(v - rv) / np.abs(rv).max()
        print(f"  p{which} l{l}: max {e.max():.2e} p99 {np.percentile(e, 99):.1e} relL2 {np.linalg.norm(v - rv) / np.linalg.norm(rv):.2e}")
