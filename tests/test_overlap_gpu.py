"""Scheme (b)/(c) overlap: turn j+1's boundary
exchange is issued on its own stream before turn j's FC compute and depends
only on the conv tops and on turn j-1 releasing its (double-buffered) slot, so
it runs UNDER turn j's FC GEMMs; turn j's gradient return likewise runs under
turn j+1's FC compute. Checked on the step's captured CUDA graph itself: tagged
marker kernels bracket each exchange, FC turn and return
(hp_cluster_debug_marker_graph), and the dependency DAG must order neither
before the other. Parity of the overlapped schedule is the scheme tests in
test_step_gpu.py (A/B/C at K=2,3,4, exact and variable)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1404_5997_b200 as hp  # noqa: E402


@pytest.mark.parametrize("K,scheme,var", [(2, "B", False), (4, "C", True), (3, "B", True), (4, "C", False)])
def test_exchange_of_next_turn_overlaps_fc_compute(K, scheme, var):
    spec = hp.tiny_cnn()
    b = 12 if K == 3 else 16
    g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.from_string(scheme),
                                          variable_batch=var, seed=1, math_mode=hp.MathMode.BF16))
    xs, ts = zip(*[hp.synthetic_batch(spec, b, worker=w) for w in range(K)])
    hpp = hp.HyperParams(lr=0.01)
    g.run_step(list(xs), list(ts), hpp)
    before = [g.param(0, 0, l) for l in range(3)]
    tags, reach = g.marker_graph(list(xs), list(ts), hpp)
    assert all(np.array_equal(a, g.param(0, 0, l)) for l, a in enumerate(before))  # captured, never run
    T = {t: i for i, t in enumerate(tags)}
    for j in range(K):
        for base in (100, 200, 300, 400, 500, 600):
            assert base + j in T, (base + j, tags)
    R = lambda a, b: bool(reach[T[a], T[b]])
    for j in range(K):
        # program order inside each stream
        assert R(100 + j, 200 + j) and R(300 + j, 400 + j) and R(500 + j, 600 + j)
        # turn j's FC compute needs its exchange; its return needs its FC dgrad
        assert R(200 + j, 300 + j) and R(300 + j, 500 + j)
        if j + 1 < K:
            # turn j+1's exchange is concurrent with turn j's FC compute
            assert not R(300 + j, 100 + j + 1) and not R(300 + j, 200 + j + 1)
            assert not R(100 + j + 1, 400 + j) and not R(200 + j + 1, 400 + j)
            # turn j's return is concurrent with turn j+1's FC compute
            assert not R(300 + j + 1, 500 + j) and not R(500 + j, 400 + j + 1)
            assert not R(600 + j, 300 + j + 1)
        if 1 <= j and j + 1 < K:
            # the exchange of turn j+1 reuses turn j-1's slot: it follows turn j-1's FC work
            assert R(300 + j - 1, 100 + j + 1)


def test_scheme_a_single_turn_graph():
    """Scheme A has one exchange (all-gather) and one return per step."""
    spec = hp.tiny_cnn()
    g = hp.Cluster(spec, hp.ClusterConfig(workers=2, per_worker_batch=8, scheme=hp.Scheme.A, seed=1,
                                          math_mode=hp.MathMode.BF16))
    xs, ts = zip(*[hp.synthetic_batch(spec, 8, worker=w) for w in range(2)])
    g.run_step(list(xs), list(ts), hp.HyperParams(lr=0.01))
    tags, reach = g.marker_graph(list(xs), list(ts), hp.HyperParams(lr=0.01))
    assert sorted(tags) == [100, 200, 300, 400, 500, 600]


def test_sliced_last_conv_matches_unsliced(monkeypatch):
    """The micro-pipelined schedule computes the same step: AlexNet K=2 scheme C
    variable, bf16, sliced vs unsliced -- the conv is the same per-image
    computation, so the parameters after the step are bit-identical."""
    spec = hp.alexnet_1col()
    K, b = 2, 4
    xs, ts = zip(*[hp.synthetic_batch(spec, b, worker=w) for w in range(K)])
    out = []
    for sliced in ("0", "1"):
        monkeypatch.setenv("HP_SLICE_LAST_CONV", sliced)
        g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.C, variable_batch=True,
                                              seed=1, math_mode=hp.MathMode.BF16))
        r = g.run_step(list(xs), list(ts), hp.HyperParams(lr=1e-3))
        out.append((r.metrics.loss, [g.param(w, which, l) for w in range(K) for which in range(8)
                                     for l in range(5 if (which & 3) < 2 else 3)]))
    assert out[0][0] == out[1][0]
    assert all(np.array_equal(a, c) for a, c in zip(out[0][1], out[1][1]))


def test_alexnet_k8_scheme_c_variable_runs():
    """configs[3] functional on one B200: AlexNet-1col b=128 per worker, K=8
    logical workers, scheme C (16-example slices), approximate variant (8 FC
    updates per step). Loss ~ L ln2 at init, 8 FC updates, replicas identical,
    integer byte counters equal the host accounting."""
    spec = hp.alexnet_1col()
    K, b = 8, 128
    cfg = hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.C, variable_batch=True, seed=1,
                           math_mode=hp.MathMode.BF16)
    g = hp.Cluster(spec, cfg)
    xs, ts = zip(*[hp.synthetic_batch(spec, b, worker=w) for w in range(K)])
    r = g.run_step(list(xs), list(ts), hp.HyperParams(lr=1e-4, weight_decay=5e-4))
    assert abs(r.metrics.loss - 1000 * np.log(2)) < 1.0
    assert r.metrics.fc_update_count == K and r.metrics.conv_update_count == 1
    bs, trace, _ = hp.step_accounting(spec, cfg)
    assert list(r.metrics.bytes_sent) == bs
    # conv_fwd, (fc_fwd j, fc_bwd j) x K, conv_bwd, sync -- the host accounting's events
    assert [(e.phase, e.sub_batch, e.worker, e.bytes_total, e.bytes_max_sender) for e in r.trace] == trace
    assert len(r.trace) == 3 + 2 * K
    for w in range(1, K):
        assert np.array_equal(g.param(w, 0, 4), g.param(0, 0, 4))


@pytest.mark.parametrize("K", [2, 4])
def test_scheme_c_turn0_exchange_overlaps_last_conv(K, monkeypatch):
    """Scheme C micro-pipelining: the last conv layer and its
    pool run in K image slices in turn order (markers 700 + j after slice j),
    and turn j's slice exchange waits for slice j only -- so turn 0's exchange
    runs under the conv of slices 1..K-1, where without slicing it waited for
    the whole conv forward. Opt-in (HP_SLICE_LAST_CONV=1): at b = 128 on B200 the
    slices' wave quantisation costs more than the exchange it hides."""
    monkeypatch.setenv("HP_SLICE_LAST_CONV", "1")
    spec = hp.alexnet_1col()
    b = 2 * K
    g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.C, variable_batch=True,
                                          seed=1, math_mode=hp.MathMode.BF16))
    xs, ts = zip(*[hp.synthetic_batch(spec, b, worker=w) for w in range(K)])
    hpp = hp.HyperParams(lr=1e-4)
    g.run_step(list(xs), list(ts), hpp)
    tags, reach = g.marker_graph(list(xs), list(ts), hpp)
    T = {t: i for i, t in enumerate(tags)}
    R = lambda a, b_: bool(reach[T[a], T[b_]])
    for j in range(K):
        assert 700 + j in T, tags
        assert R(700 + j, 100 + j)                # turn j's exchange needs slice j
        assert R(700 + K - 1, 300 + j)            # the FC compute follows the whole conv (stream order)
        if j + 1 < K:
            assert R(700 + j, 700 + j + 1)
        if j <= 1:
            # turns 0 and 1 exchange into fresh slots: they wait for their own slice, not the later
            # ones (turn j >= 2 reuses turn j-2's slot and so follows its FC work, after the conv)
            for later in range(j + 1, K):
                assert not R(700 + later, 100 + j) and not R(700 + later, 200 + j), (j, later)
