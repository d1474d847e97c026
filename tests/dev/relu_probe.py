"""Dev: last-fc-layer ReLU across schemes / steps / graphs vs the oracle (prints)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
import paper_1404_5997_b200 as hp
from helpers import rel_err


def run(K, scheme, var, steps, graphs, relu_last=True, ws=30.0, b=8, math=hp.MathMode.F32X3, lr=0.001):
    spec = hp.tiny_cnn()
    spec.fc_layers[-1].relu = relu_last
    g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.from_string(scheme),
                                          variable_batch=var, seed=1, math_mode=math))
    g.set_graphs(graphs)
    o = O.OracleCluster(spec, workers=K, per_worker_batch=b, scheme=scheme, variable_batch=var, precision="single", seed=1)
    for w in range(K):
        for which in (0, 2):
            for l in range(3 if which == 0 else 2):
                a = g.param(w, which, l)
                g.write_param(w, which, l, a * ws)
                o.write_param(w, which, l, (a * ws).astype(np.float64))
    for s in range(steps):
        xs, ts = zip(*[hp.synthetic_batch(spec, b, step=s, worker=w) for w in range(K)])
        r = g.run_step(list(xs), list(ts), hp.HyperParams(momentum=0.9, lr=lr, weight_decay=5e-4))
        m = o.run_step([x.astype(np.float64) for x in xs], [t.astype(np.float64) for t in ts], O.make_hyper_c(0.9, lr, 5e-4))
    errs = {(which, l): rel_err(g.param(0, which, l), o.param(0, which, l)) for which in (4, 5, 6, 7) for l in range(3 if which < 6 else 2)}
    worst = max(errs.values())
    print(f"K={K} {scheme} var={var} ws={ws} lr={lr} steps={steps} graphs={graphs} relu_last={relu_last}: loss {r.metrics.loss:.6f}/{m.loss:.6f} worst {worst:.2e}",
          {k: f"{v:.1e}" for k, v in errs.items() if v > 1e-4})


if __name__ == '__main__':
  for K, sc, var in [(2, "A", False), (2, "B", False), (2, "C", False), (2, "C", True), (4, "B", False)]:
    for steps in (1, 2):
        run(K, sc, var, steps, False)
    run(K, sc, var, 2, True)
  run(2, "C", False, 1, False, relu_last=False)
