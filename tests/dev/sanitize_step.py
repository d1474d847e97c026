"""Dev: one small eager step per configuration for compute-sanitizer runs
(memcheck / racecheck / synccheck over every kernel of the step, the tcgen05 /
TMA / mbarrier GEMMs included). argv[1]: tiny | tiny_bf16 | alexnet."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1404_5997_b200 as hp

which = sys.argv[1] if len(sys.argv) > 1 else "tiny"
if which == "alexnet":
    spec, K, b, math, scheme = hp.alexnet_1col(), 2, 4, hp.MathMode.BF16, hp.Scheme.C
elif which == "tiny_bf16":
    spec, K, b, math, scheme = hp.tiny_cnn(), 2, 8, hp.MathMode.BF16, hp.Scheme.B
else:
    spec, K, b, math, scheme = hp.tiny_cnn(), 2, 8, hp.MathMode.F32X3, hp.Scheme.C
c = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=scheme, seed=1, math_mode=math,
                                      variable_batch=scheme == hp.Scheme.C))
c.set_graphs(False)
xs, ts = zip(*[hp.synthetic_batch(spec, b, worker=w) for w in range(K)])
r = c.run_step(list(xs), list(ts), hp.HyperParams(lr=0.01))
print(which, "loss", r.metrics.loss, "launches", c.last_step_launches())
