"""Dev: per-tensor error report of the AlexNet b=128 first step vs the committed
double-oracle fixture, across math modes / kernel toggles; and the tiny-CNN
last-layer-ReLU case vs the oracle. Prints, asserts nothing."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_1404_5997_b200 as hp  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden", "alexnet_step1.npz")
SAMPLE, PRIME = 131072, 2654435761


def sample_index(n):
    if n <= SAMPLE:
        return np.arange(n, dtype=np.int64)
    return (np.arange(SAMPLE, dtype=np.int64) * PRIME) % n


def alexnet(case, math, shift=True):
    gold = np.load(GOLD)
    K, scheme, var = {"k1b": (1, "B", False), "k2c": (2, "C", True)}[case]
    mu, lr, wd = gold["hyper"]
    b = int(gold["b"][0])
    spec = hp.alexnet_1col()
    g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.from_string(scheme),
                                          variable_batch=var, seed=1, math_mode=math))
    if not shift:
        g.set_shift_conv(False)
    xs, ts = zip(*[hp.synthetic_batch(spec, b, step=0, worker=w) for w in range(K)])
    r = g.run_step(list(xs), list(ts), hp.HyperParams(momentum=mu, lr=lr, weight_decay=wd))
    lo = float(gold[f"{case}_loss"][0])
    print(f"== {case} {math.name} shift={shift}: loss {r.metrics.loss:.8f} oracle {lo:.8f} rel {abs(r.metrics.loss-lo)/lo:.2e}")
    for w in range(K):
        for which in (4, 5, 6, 7):
            for l in range(len(spec.conv_layers) if which in (4, 5) else len(spec.fc_layers)):
                if which in (4, 5) and w > 0:
                    continue
                key = f"{case}_w{w}_p{which}_l{l}"
                v = g.param(w, which, l)
                idx = sample_index(v.size)
                ref, mx = gold[key + "_val"].astype(np.float64), float(gold[key + "_max"][0])
                d = np.abs(v[idx].astype(np.float64) - ref)
                e = d.max() / mx
                em = abs(np.abs(v).max() - mx) / mx
                worst = idx[int(d.argmax())]
                print(f"  w{w} p{which} l{l}: n={v.size} err {e:.3e} maxerr {em:.3e} rms {np.sqrt((d**2).mean())/mx:.3e}"
                      f" worst@{worst} gpu {v[worst]:.4e} ref {ref[int(d.argmax())]:.4e} max {mx:.4e}")
    return g


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("all", "alex"):
        alexnet("k1b", hp.MathMode.BF16)
        alexnet("k1b", hp.MathMode.BF16, shift=False)
        alexnet("k1b", hp.MathMode.F32X3)
        alexnet("k2c", hp.MathMode.BF16)
    if what in ("all", "relu"):
        os.environ["HP_TOL_REPORT"] = "1"
        import test_step_gpu as T
        spec = hp.tiny_cnn()
        spec.fc_layers[-1].relu = True
        for args in [dict(K=2, scheme="C", wscale=30.0, lr=0.001, b=8, steps=2),
                     dict(K=1, scheme="B", wscale=30.0, lr=0.001, b=8, steps=2),
                     dict(K=1, scheme="B", wscale=1.0, lr=0.001, b=8, steps=1)]:
            print("== relu", args)
            try:
                T.compare(spec, args["K"], args["scheme"], False, hp.MathMode.F32X3, args["b"], steps=args["steps"],
                          lr=args["lr"], wscale=args["wscale"])
            except AssertionError as ex:
                print("   FAIL", ex)
        spec.fc_layers[-1].relu = False
        print("== norelu ws30 K=1")
        try:
            T.compare(spec, 1, "B", False, hp.MathMode.F32X3, 8, steps=2, lr=0.001, wscale=30.0)
        except AssertionError as ex:
            print("   FAIL", ex)
