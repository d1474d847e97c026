"""Dev: AlexNet bf16 step vs the bf16-storage oracle, error distributions per
tensor under kernel toggles (prints)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
import paper_1404_5997_b200 as hp

spec = hp.alexnet_1col()
b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
lr = 0.01
xs, ts = hp.synthetic_batch(spec, b, step=0, worker=0)
o = O.OracleCluster(spec, workers=1, per_worker_batch=b, scheme="B", precision="single", seed=1)
o.set_storage_rounding("bf16")
m = o.run_step([xs.astype(np.float64)], [ts.astype(np.float64)], O.make_hyper_c(0.9, lr, 5e-4))
ref = {(which, l): o.param(0, which, l) for which in (4, 5, 6, 7) for l in range(5 if which < 6 else 3)}


def go(name, **tog):
    g = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=b, scheme=hp.Scheme.B, seed=1,
                                          math_mode=hp.MathMode.BF16))
    for k, v in tog.items():
        getattr(g, "set_" + k)(v)
    r = g.run_step([xs], [ts], hp.HyperParams(momentum=0.9, lr=lr, weight_decay=5e-4))
    print(f"== {name}: loss {r.metrics.loss:.8f} / {m.loss:.8f}")
    for (which, l), rv in ref.items():
        v = g.param(0, which, l).astype(np.float64)
        e = np.abs(v - rv) / np.abs(rv).max()
        q = np.percentile(e, [50, 90, 99, 99.9])
        print(f"  p{which} l{l}: max {e.max():.2e} p50 {q[0]:.1e} p90 {q[1]:.1e} p99 {q[2]:.1e} p99.9 {q[3]:.1e} n>1e-2 {int((e > 1e-2).sum())}/{e.size}")


go("default")
go("no-graphs", graphs=False)
go("unfused-sgd", fuse_fc_sgd=False, graphs=False)
go("no-shift", shift_conv=False, graphs=False)
