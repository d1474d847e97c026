"""Dev: bf16 GPU steps vs the oracle in double and in bf16-storage mode (prints)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
import paper_1404_5997_b200 as hp
from helpers import rel_err


def run(spec, K, scheme, var, b, steps=1, lr=0.01, name=""):
    g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.from_string(scheme),
                                          variable_batch=var, seed=1, math_mode=hp.MathMode.BF16))
    os_ = {}
    for mode in ("double", "bf16"):
        o = O.OracleCluster(spec, workers=K, per_worker_batch=b, scheme=scheme, variable_batch=var, precision="single", seed=1)
        o.set_storage_rounding(mode)
        os_[mode] = o
    for s in range(steps):
        xs, ts = zip(*[hp.synthetic_batch(spec, b, step=s, worker=w) for w in range(K)])
        r = g.run_step(list(xs), list(ts), hp.HyperParams(momentum=0.9, lr=lr, weight_decay=5e-4))
        ms = {k: o.run_step([x.astype(np.float64) for x in xs], [t.astype(np.float64) for t in ts], O.make_hyper_c(0.9, lr, 5e-4)) for k, o in os_.items()}
    nl = lambda which: len(spec.conv_layers) if (which & 3) < 2 else len(spec.fc_layers)
    for k, o in os_.items():
        errs = {(w, which, l): rel_err(g.param(w, which, l), o.param(w, which, l)) for w in range(K) for which in (4, 5, 6, 7) for l in range(nl(which))}
        print(f"{name} K={K} {scheme} var={var} b={b} steps={steps} vs {k}: loss {r.metrics.loss:.8f}/{ms[k].loss:.8f} worst {max(errs.values()):.2e}",
              " ".join(f"{w}{which}{l}:{v:.1e}" for (w, which, l), v in errs.items()), flush=True)


if __name__ == "__main__":
    for a in sys.argv[1:] or ["tiny", "alex"]:
        if a == "tiny":
            run(hp.tiny_cnn(), 1, "B", False, 32, name="tiny")
            run(hp.tiny_cnn(), 2, "A", False, 128, steps=2, name="tiny")
        else:
            run(hp.alexnet_1col(), 1, "B", False, 16, name="alex")
            run(hp.alexnet_1col(), 2, "C", True, 8, name="alex")
