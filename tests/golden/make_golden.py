"""Generate golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run here, where /root/reference exists (`make -C oracle ref` first). Writes
tests/golden/reference_golden.npz, which the CPU and GPU suites check the C
restatement against on machines without the reference (the GPU box).
"""
import os
import sys
import types

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402


def toy_spec():
    c = lambda i, o, k, s=1, p=0: types.SimpleNamespace(in_channels=i, out_channels=o, kernel=k, stride=s, pad=p, relu=True)
    f = lambda i, o, r=False: types.SimpleNamespace(in_dim=i, out_dim=o, relu=r)
    # SPEC.md toy spec: 2x6x6; conv 2->3 k3 p1, 3->4 k2 s2; fc 36->8 ReLU, 8->4
    return types.SimpleNamespace(conv_layers=[c(2, 3, 3, 1, 1), c(3, 4, 2, 2, 0)],
                                 fc_layers=[f(36, 8, True), f(8, 4)], input_shape=[2, 6, 6], num_classes=4)


CASES = [  # (K, scheme, variable, precision)
    (1, "B", False, "double"), (2, "A", False, "double"), (2, "B", True, "double"),
    (4, "C", False, "double"), (4, "C", True, "double"), (4, "B", False, "single"),
]


def main():
    assert O.ref_available(), "build the reference first: make -C oracle ref"
    out = {}
    out["gauss_seed0"] = np.array([0.0])
    g = np.empty(64)
    lib = O.ref_lib()
    lib.ref_gaussian_fill(0, O._dp(g), 64)
    out["gauss_seed0"] = g.copy()
    lib.ref_gaussian_fill(12345, O._dp(g), 64)
    out["gauss_seed12345"] = g.copy()
    spec = toy_spec()
    rng = np.random.default_rng(7)
    for ci, (K, scheme, var, prec) in enumerate(CASES):
        b = 4
        r = O.RefCluster(spec, workers=K, per_worker_batch=b, scheme=scheme, variable_batch=var, precision=prec, seed=3)
        for w in range(K):  # scale weights so ReLUs are active
            for which in (0, 2):
                for l in range(2):
                    r.write_param(w, which, l, r.param(w, which, l) * 30.0)
        hp = O.make_hyper_c(0.9, 0.05, 5e-4)
        losses = []
        for s in range(3):
            xs = [rng.normal(size=(b, 2, 6, 6)) for _ in range(K)]
            ts = [np.eye(4)[rng.integers(0, 4, size=b)] for _ in range(K)]
            for w in range(K):
                out[f"c{ci}_s{s}_x{w}"] = xs[w]
                out[f"c{ci}_s{s}_t{w}"] = ts[w]
            m = r.run_step(xs, ts, hp)
            losses.append(m.loss)
            out[f"c{ci}_s{s}_bytes"] = np.array(list(m.bytes_sent), dtype=np.int64)
            out[f"c{ci}_s{s}_trace"] = np.array(r.trace(), dtype=np.int64)
        out[f"c{ci}_loss"] = np.array(losses)
        for w in range(K):
            for which in range(8):
                for l in range(2):
                    out[f"c{ci}_w{w}_p{which}_l{l}"] = r.param(w, which, l)
    out["cases"] = np.array([(K, "ABC".index(s), int(v), 0 if p == "single" else 1) for K, s, v, p in CASES])
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
