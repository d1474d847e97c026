"""The BENCHMARKED configuration against the double oracle.

bench.py times AlexNet-1col, b=128 per GPU, bf16, scheme B exact SGD (configs[2]
at N=1). These tests run exactly that step -- same cluster config, so the same
kernel and plan choices: space-to-depth conv1 on TMA im2col, the flat-shift
conv2-5 fprop/dgrad over q-layout activations with RowMap epilogues, the flat
LRN+pool kernels, the split-K plans of b=128 -- plus configs[3]'s mode (scheme C,
approximate/variable FC update) at K=2 on the logical transport, and compare
every parameter tensor's momentum after the first step (pure gradient history,
-lr*(g + wd*w0), the paper's mu/lr/wd) and the loss with the oracle's double
step on identical inputs (tests/golden/make_alexnet_golden.py, committed
fixture: full-tensor max|.| plus a fixed sample of entries per tensor).

Tolerance (bf16 operands, fp32 accumulate): max |gpu - oracle| /
max |oracle| <= 3e-2 per tensor over the sampled entries, and the tensor's
max |.| within 3e-2; loss within 1e-4 relative.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1404_5997_b200 as hp  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "alexnet_step1.npz")
TOL = 3e-2
CASES = {"k1b": (1, "B", False), "k2c": (2, "C", True)}
SAMPLE, PRIME = 131072, 2654435761


def sample_index(n):
    if n <= SAMPLE:
        return np.arange(n, dtype=np.int64)
    return (np.arange(SAMPLE, dtype=np.int64) * PRIME) % n


@pytest.mark.parametrize("case", list(CASES))
def test_alexnet_bf16_first_step_matches_oracle(case):
    gold = np.load(GOLD)
    if f"{case}_loss" not in gold:
        pytest.fail(f"fixture {case} missing: run tests/golden/make_alexnet_golden.py")
    K, scheme, var = CASES[case]
    mu, lr, wd = gold["hyper"]
    b = int(gold["b"][0])
    spec = hp.alexnet_1col()
    g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.from_string(scheme),
                                          variable_batch=var, seed=1, math_mode=hp.MathMode.BF16))
    xs, ts = zip(*[hp.synthetic_batch(spec, b, step=0, worker=w) for w in range(K)])
    r = g.run_step(list(xs), list(ts), hp.HyperParams(momentum=mu, lr=lr, weight_decay=wd))
    lo = float(gold[f"{case}_loss"][0])
    assert abs(r.metrics.loss - lo) <= 1e-4 * abs(lo), (r.metrics.loss, lo)
    worst = {}
    for w in range(K):
        for which in (4, 5, 6, 7):
            for l in range(len(spec.conv_layers) if which in (4, 5) else len(spec.fc_layers)):
                key = f"{case}_w{w if which in (6, 7) else 0}_p{which}_l{l}"
                v = g.param(w, which, l)
                assert v.size == int(gold[key + "_n"][0])
                ref, mx = gold[key + "_val"].astype(np.float64), float(gold[key + "_max"][0])
                e = np.abs(v[sample_index(v.size)].astype(np.float64) - ref).max() / mx
                em = abs(np.abs(v).max() - mx) / mx
                worst[(w, which, l)] = (e, em)
                assert e <= TOL and em <= TOL, (w, which, l, e, em)
    # conv replicas identical after the all-reduce
    for w in range(1, K):
        for l in range(len(spec.conv_layers)):
            assert np.array_equal(g.param(w, 0, l), g.param(0, 0, l))
    print({k: tuple(round(x, 5) for x in v) for k, v in worst.items()})
