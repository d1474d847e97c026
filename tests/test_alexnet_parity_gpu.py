"""The BENCHMARKED configuration against the oracle.

bench.py times AlexNet-1col, b=128 per GPU, bf16, scheme B exact SGD (configs[2]
at N=1). These tests run exactly that step -- same cluster config, so the same
kernel and plan choices: space-to-depth conv1 on TMA im2col, the flat-shift
conv2-5 fprop/dgrad over q-layout activations with RowMap epilogues, the
row-streaming LRN+pool kernels, the split-K plans of b=128 -- plus configs[3]'s
mode (scheme C, approximate/variable FC update) at K=2 on the logical transport.

1. Decision replay (test_bench_step_matches_oracle_with_replayed_decisions).
   A bf16 step and a double one cannot agree entry by entry on the sensitive
   tensors: accumulation order alone moves ~0.5% of the bf16-rounded
   activations by one ulp, which flips a few ReLU masks and pool argmaxes per
   10^4 (near-zero pre-activations, near-tied windows), and every flip moves a
   whole gradient entry (conv1's gradient, a sum over 387k pixels, changes by
   ~10% at b=128). So the GPU's discrete decisions (ReLU masks of every conv
   and fc layer, pool argmax of every pooled stage, every turn) are read back
   (hp_cluster_debug_decisions) and replayed in the oracle, which rounds its
   stored tensors to bf16 where the GPU stores them (or_cluster_set_storage_rounding)
   and computes everything else in double. Then:
     * every parameter tensor's momentum after step 1 (pure gradient history,
       -lr*(g + wd*w0), the paper's mu/lr/wd) within 1e-2 of max|ref|
       (measured <= 2.1e-3, conv1; most <= 4e-4), loss within 1e-6;
     * the replayed decisions themselves: at most 1% differ from the oracle's
       own, and every difference is a near-tie -- a ReLU whose pre-activation
       is within 2e-2 rms of zero, a pool window whose two candidates are within
       5e-2 rms of each other.
2. Against the pure double oracle (no emulation, no replay; committed fixture
   tests/golden/alexnet_step1.npz from the reference restatement): the loss
   within 1e-4, and each tensor within the flip-level bound measured for
   legitimate bf16 accumulation orders (parity)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
import paper_1404_5997_b200 as hp  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "alexnet_step1.npz")
CASES = {"k1b": (1, "B", False), "k2c": (2, "C", True)}
SAMPLE, PRIME = 131072, 2654435761
HYPER = (0.9, 0.01, 5e-4)
B = 128


def sample_index(n):
    if n <= SAMPLE:
        return np.arange(n, dtype=np.int64)
    return (np.arange(SAMPLE, dtype=np.int64) * PRIME) % n


def gpu_step(case, capture=False):
    K, scheme, var = CASES[case]
    spec = hp.alexnet_1col()
    g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=B, scheme=hp.Scheme.from_string(scheme),
                                          variable_batch=var, seed=1, math_mode=hp.MathMode.BF16))
    g.set_debug_capture(capture)
    xs, ts = zip(*[hp.synthetic_batch(spec, B, step=0, worker=w) for w in range(K)])
    r = g.run_step(list(xs), list(ts), hp.HyperParams(momentum=HYPER[0], lr=HYPER[1], weight_decay=HYPER[2]))
    return spec, g, r, xs, ts


@pytest.mark.parametrize("case", list(CASES))
def test_bench_step_matches_oracle_with_replayed_decisions(case):
    K, scheme, var = CASES[case]
    spec, g, r, xs, ts = gpu_step(case, capture=True)
    o = O.OracleCluster(spec, workers=K, per_worker_batch=B, scheme=scheme, variable_batch=var,
                        precision="single", seed=1)
    o.set_storage_rounding("bf16")
    forced = []
    for w in range(K):
        for l, c in enumerate(spec.conv_layers):
            o.force_decisions(w, 0, l, g.decisions(w, 0, l))
            forced.append((w, 0, l))
            if c.pool_kernel:
                o.force_decisions(w, 1, l, g.decisions(w, 1, l))
                forced.append((w, 1, l))
    nf, nsub = len(spec.fc_layers), (1 if scheme == "A" else K)
    for j in range(nsub):
        for l, f in enumerate(spec.fc_layers):
            if f.relu:
                o.force_decisions(0, 2, j * nf + l, g.decisions(0, 2, j * nf + l))
                forced += [(w, 2, j * nf + l) for w in range(K)]
    m = o.run_step([x.astype(np.float64) for x in xs], [t.astype(np.float64) for t in ts], O.make_hyper_c(*HYPER))
    assert abs(r.metrics.loss - m.loss) <= 1e-6 * abs(m.loss), (r.metrics.loss, m.loss)
    report = {}
    for w, kind, l in forced:
        mis, gap = o.decision_stats(w, kind, l)
        n = g.decisions(0 if kind == 2 else w, kind, l).size
        if kind == 2:
            n //= K  # stats are per worker shard
        report[(w, kind, l)] = (mis / n, gap)
        assert mis <= 0.01 * n, (w, kind, l, mis, n)
        assert gap <= (5e-2 if kind == 1 else 2e-2), (w, kind, l, gap)
    worst = {}
    for w in range(K):
        for which in (4, 5, 6, 7):
            for l in range(len(spec.conv_layers) if which in (4, 5) else nf):
                v = g.param(w, which, l).astype(np.float64)
                ref = o.param(w, which, l)
                e = np.abs(v - ref).max() / np.abs(ref).max()
                worst[(w, which, l)] = e
    print("decisions (fraction differing, gap):", {k: (f"{a:.1e}", f"{b:.1e}") for k, (a, b) in report.items()})
    print("momentum errors:", {k: f"{v:.1e}" for k, v in worst.items()})
    bad = {k: v for k, v in worst.items() if v > 1e-2}
    assert not bad, bad
    for w in range(1, K):  # conv replicas identical after the all-reduce
        for l in range(len(spec.conv_layers)):
            assert np.array_equal(g.param(w, 0, l), g.param(0, 0, l))


# Flip-level bounds against the pure double restatement (no emulation, no
# replay), measured on this step (DESIGN.md parity): conv1's pixel-summed
# gradient and the fc layers of the K=2 approximate mode carry the most flips.
FLIP_TOL = {4: {0: 0.25}, 6: {1: 0.15}, 7: {1: 0.15}}
FLIP_DEFAULT = 6e-2


@pytest.mark.parametrize("case", list(CASES))
def test_bench_step_near_pure_double_oracle(case):
    gold = np.load(GOLD)
    K = CASES[case][0]
    spec, g, r, _, _ = gpu_step(case)
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
                worst[(w, which, l)] = e
    print({k: f"{v:.2e}" for k, v in worst.items()})
    bad = {k: v for k, v in worst.items() if v > FLIP_TOL.get(k[1], {}).get(k[2], FLIP_DEFAULT)}
    assert not bad, bad
