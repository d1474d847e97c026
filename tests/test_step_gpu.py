"""Step parity: the B200 run_step (C ABI) against the CPU oracle on identical
inputs and seeds. The oracle restates the reference in double (pinned
bit-exactly to the compiled reference in tests/test_oracle_vs_reference.py).

Tolerances (stated; max |gpu - oracle| / max |oracle| per parameter tensor
after the steps, weights and momenta; loss relative):
  f32x3 (3xTF32, parity mode):   momenta/biases 2e-3, weights 2e-5, loss 2e-5
  f32x3, mask-stable setup (test_active_relus, weights x30):  everything 3e-5
                                 (measured <= 1.6e-5; the reference's own
                                 FP32-vs-FP64 gap is up to 6.9e-6)
  tf32:                          momenta 8e-2, weights 1e-4, loss 1e-5
  bf16 with decision replay:     momenta/biases 3e-2, weights 5e-4, loss 1e-4
(momenta and biases -- zero at init -- are pure gradient history after two
steps, so they carry the GEMM input rounding undiluted and use the first
tolerance; weights use the second. The f32x3 gradient tolerance at the
0.01-sigma init is set by ReLU mask flips, not GEMM accuracy: many
pre-activations sit within fp32 error of zero, and conv1's gradient collects
every flip below it. In bf16 a flip is the rule, not the exception, so the bf16
cases replay the GPU's discrete decisions (ReLU masks, per step and per turn)
in the oracle, which also rounds its stored tensors to bf16 where the GPU
stores them -- the method of tests/test_alexnet_parity_gpu.py.)
Integer outputs (byte counters, trace, update counts) must be identical."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
import paper_1404_5997_b200 as hp  # noqa: E402
from helpers import rel_err  # noqa: E402

TOL = {hp.MathMode.F32X3: (2e-3, 2e-5, 2e-5), hp.MathMode.TF32: (8e-2, 1e-4, 1e-5),
       hp.MathMode.BF16: (3e-2, 5e-4, 1e-4)}
TOL_STABLE = (3e-5, 3e-5, 2e-5)  # f32x3, no mask flips (weights x30)


def replay_decisions(spec, K, scheme, g, o):
    """Force the GPU's last-step ReLU masks (conv, and fc per turn) into the
    oracle's next step (hp_cluster_debug_decisions / or_cluster_force_decisions)."""
    for w in range(K):
        for l, c in enumerate(spec.conv_layers):
            if c.relu:
                o.force_decisions(w, 0, l, g.decisions(w, 0, l))
            if c.pool_kernel:
                o.force_decisions(w, 1, l, g.decisions(w, 1, l))
    nf, nsub = len(spec.fc_layers), (1 if scheme == "A" else K)
    for j in range(nsub):
        for l, f in enumerate(spec.fc_layers):
            if f.relu:
                o.force_decisions(0, 2, j * nf + l, g.decisions(0, 2, j * nf + l))


def compare(spec, K, scheme, var, math, b, steps=2, lr=0.05, wscale=1.0, seed=1, skip=False, tol=None):
    cfg = hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.from_string(scheme),
                           variable_batch=var, seed=seed, math_mode=math)
    g = hp.Cluster(spec, cfg)
    o = O.OracleCluster(spec, workers=K, per_worker_batch=b, scheme=scheme, variable_batch=var,
                        precision="single", seed=seed)
    if skip:
        g.set_skip_sync_broadcast(True)
        o.set_skip_sync_broadcast(True)
    replay = math == hp.MathMode.BF16
    if replay:
        g.set_debug_capture(True)
        o.set_storage_rounding("bf16")
    nl = lambda which: len(spec.conv_layers) if (which & 3) < 2 else len(spec.fc_layers)
    for w in range(K):  # identical initial parameters (GaussianSampler replay + layout permutations)
        for which in range(4):
            for l in range(nl(which)):
                a = g.param(w, which, l)
                assert np.array_equal(a.astype(np.float64), o.param(w, which, l))
                if wscale != 1.0 and which in (0, 2):
                    g.write_param(w, which, l, a * wscale)
                    o.write_param(w, which, l, (a * wscale).astype(np.float64))
    hpg = hp.HyperParams(momentum=0.9, lr=lr, weight_decay=5e-4)
    hpo = O.make_hyper_c(0.9, lr, 5e-4)
    mt, wt, lt = tol or TOL[math]
    for s in range(steps):
        xs, ts = zip(*[hp.synthetic_batch(spec, b, step=s, worker=w) for w in range(K)])
        r = g.run_step(list(xs), list(ts), hpg)
        if replay:
            replay_decisions(spec, K, scheme, g, o)
        m = o.run_step([x.astype(np.float64) for x in xs], [t.astype(np.float64) for t in ts], hpo)
        assert abs(r.metrics.loss - m.loss) <= lt * abs(m.loss), (r.metrics.loss, m.loss)
        assert list(r.metrics.bytes_sent) == list(m.bytes_sent)
        assert [(e.phase, e.sub_batch, e.worker, e.bytes_total, e.bytes_max_sender) for e in r.trace] == o.trace()
        assert r.metrics.fc_update_count == m.fc_update_count
        assert r.metrics.conv_update_count == m.conv_update_count
    bad = []
    for w in range(K):
        assert g.worker_bytes(w) == o.worker_bytes(w)
        for which in range(8):
            for l in range(nl(which)):
                e = rel_err(g.param(w, which, l), o.param(w, which, l))
                if os.environ.get("HP_TOL_REPORT"):
                    print(f"TOL {math.name} K={K} {scheme} var={var} b={b} ws={wscale} w{w} p{which} l{l} {e:.3e}")
                # biases start at zero, so (like momenta) they are pure gradient history
                if e > (mt if (which >= 4 or which in (1, 3)) else wt):
                    bad.append((w, which, l, e))
    assert not bad, bad
    # replica consistency: conv replicas identical across workers (unless the
    # negative control skipped the broadcast)
    for w in range(1, K):
        for l in range(len(spec.conv_layers)):
            assert np.array_equal(g.param(w, 0, l), g.param(0, 0, l)) != skip
    # gathered_model (cluster.cpp:417-437): worker 0's conv replica + the fc
    # shards pasted back by column -- exactly the per-worker tensors compared above
    (gconv, gfc) = g.gathered_model()
    for l, (k, b_) in enumerate(gconv):
        assert np.array_equal(k.ravel(), g.param(0, 0, l)) and np.array_equal(b_, g.param(0, 1, l))
    for l, (wm, b_) in enumerate(gfc):
        fin = spec.fc_layers[l].in_dim
        assert np.array_equal(wm, np.concatenate([g.param(w, 2, l).reshape(fin, -1) for w in range(K)], axis=1))
        assert np.array_equal(b_, np.concatenate([g.param(w, 3, l) for w in range(K)]))
    return g, o


@pytest.mark.parametrize("math", [hp.MathMode.F32X3, hp.MathMode.TF32, hp.MathMode.BF16])
def test_tiny_k1(math):
    """configs[0]: tiny CNN, K=1 (b=32 here for time; b=128 in test_tiny_configs)."""
    compare(hp.tiny_cnn(), 1, "B", False, math, 32)


@pytest.mark.parametrize("K,scheme,var", [(2, "A", False), (2, "B", False), (2, "C", True), (4, "B", True),
                                          (4, "C", False), (4, "A", False), (3, "B", False)])
def test_tiny_schemes(K, scheme, var):
    """Scheme routing, uneven fc shards (K=3: 85/85/86, K=4: 10 -> 2/2/2/4), variable mode."""
    compare(hp.tiny_cnn(), K, scheme, var, hp.MathMode.F32X3, 12 if K == 3 else 16)


@pytest.mark.parametrize("math", [hp.MathMode.F32X3, hp.MathMode.BF16])
def test_tiny_configs(math):
    """configs[0..1] at their full size: K=1 b=128, and K=2 scheme A exact b=128."""
    compare(hp.tiny_cnn(), 1, "B", False, math, 128, steps=1)
    compare(hp.tiny_cnn(), 2, "A", False, math, 128, steps=1)


def test_active_relus():
    """Weights x30 so most ReLUs are active and the gradients are large."""
    compare(hp.tiny_cnn(), 2, "C", False, hp.MathMode.F32X3, 8, steps=2, lr=0.001, wscale=30.0, tol=TOL_STABLE)


@pytest.mark.parametrize("K,scheme,var", [(1, "B", False), (2, "C", True)])
def test_alexnet_small_batch(K, scheme, var):
    """AlexNet-1col (LRN, overlapping pool, floor-mode conv1) at b=2 per worker in 3xTF32."""
    compare(hp.alexnet_1col(), K, scheme, var, hp.MathMode.F32X3, 2, steps=1, lr=0.01)


def test_last_fc_layer_relu():
    """A spec whose LAST fc layer has a ReLU: the logit gradient is masked by
    relu_backward(pre, grad) (model.cpp:302, cluster.cpp:569) before the fc
    backward and the boundary return."""
    spec = hp.tiny_cnn()
    spec.fc_layers[-1].relu = True
    # weights x10: logits well away from 0 (x30 makes step 2 chaotic -- the same
    # 1e-2 divergence appears with or without the ReLU, tests/dev/relu_probe.py)
    compare(spec, 2, "C", False, hp.MathMode.F32X3, 8, steps=2, lr=0.001, wscale=10.0)
    compare(spec, 2, "A", False, hp.MathMode.F32X3, 8, steps=2, lr=0.001, wscale=10.0)
    compare(spec, 1, "B", False, hp.MathMode.BF16, 16, steps=1)


def test_device_target_domain_error_before_any_update():
    """logistic_xent's DomainError (tensor.cpp:600-603) for DEVICE-resident
    targets is raised before the step changes any parameter or momentum."""
    import torch
    spec = hp.tiny_cnn()
    g = hp.Cluster(spec, hp.ClusterConfig(workers=2, per_worker_batch=8, scheme=hp.Scheme.B, seed=1,
                                          math_mode=hp.MathMode.BF16))
    xs, ts = zip(*[hp.synthetic_batch(spec, 8, worker=w) for w in range(2)])
    dx = [torch.from_numpy(x).cuda() for x in xs]
    dt = [torch.from_numpy(t).cuda() for t in ts]
    g.run_step(dx, dt, hp.HyperParams(lr=0.01))
    before = [g.param(w, which, l) for w in range(2) for which in range(8) for l in range(3 if (which & 3) < 2 else 2)]
    bad = dt[1].clone()
    bad[3, 2] = 1.5
    with pytest.raises(hp.DomainError, match="outside"):
        g.run_step(dx, [dt[0], bad], hp.HyperParams(lr=0.01))
    after = [g.param(w, which, l) for w in range(2) for which in range(8) for l in range(3 if (which & 3) < 2 else 2)]
    assert all(np.array_equal(a, b) for a, b in zip(before, after))
    g.run_step(dx, dt, hp.HyperParams(lr=0.01))  # still usable


def test_alexnet_bf16_loss_and_io():
    """Full AlexNet b=128 bf16 step runs; loss ~ L*ln2 at init; host inputs counted."""
    spec = hp.alexnet_1col()
    g = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=128, math_mode=hp.MathMode.BF16, seed=1))
    x, t = hp.synthetic_batch(spec, 128)
    r = g.run_step([x], [t], hp.HyperParams(lr=0.01, weight_decay=5e-4))
    assert abs(r.metrics.loss - 1000 * np.log(2)) < 1.0
    h2d, d2h = g.last_step_io()
    assert h2d == x.nbytes + t.nbytes and d2h > 0
    assert g.last_step_launches() > 20
    assert g.last_gemm_flops() > 5e11  # ~626 GFLOP algorithmic


def test_cuda_graph_replay_is_bit_identical():
    """Eager, first capture and replays produce bit-identical parameters and
    losses (every kernel is deterministic; the graph bakes the same launches)."""
    import torch
    spec = hp.tiny_cnn()
    res = []
    for graphs in (False, True):
        g = hp.Cluster(spec, hp.ClusterConfig(workers=2, per_worker_batch=16, scheme=hp.Scheme.C, seed=3,
                                              math_mode=hp.MathMode.BF16))
        g.set_graphs(graphs)
        bufs = [hp.synthetic_batch(spec, 16, step=s, worker=w) for s in range(2) for w in range(2)]
        dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()) for x, t in bufs]
        losses = []
        for s in range(6):  # each of the 2 input sets: eager, capture, replay
            k = s % 2
            xs = [dev[2 * k][0], dev[2 * k + 1][0]]
            ts = [dev[2 * k][1], dev[2 * k + 1][1]]
            losses.append(g.run_step(xs, ts, hp.HyperParams(lr=0.01)).metrics.loss)
        res.append((losses, [g.param(w, which, l) for w in range(2) for which in range(8)
                             for l in range(3 if (which & 3) < 2 else 2)]))
    assert res[0][0] == res[1][0]
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)


def test_prefetch_double_buffer_matches_plain_host_steps():
    """hp_cluster_prefetch: host batches staged on the copy stream (two slots,
    overlapping the previous step) give bit-identical results to plain host
    steps; the H2D bytes are still charged to the consuming step; a run_step
    on different host buffers ignores the staged slot."""
    import torch
    spec = hp.tiny_cnn()
    host = [hp.synthetic_batch(spec, 16, step=s, worker=w) for s in range(3) for w in range(2)]
    pinned = [(torch.from_numpy(x).pin_memory(), torch.from_numpy(t).pin_memory()) for x, t in host]
    res = []
    for pre in (False, True):
        g = hp.Cluster(spec, hp.ClusterConfig(workers=2, per_worker_batch=16, scheme=hp.Scheme.B, seed=5,
                                              math_mode=hp.MathMode.BF16))
        losses, io = [], []
        order = [0, 1, 2, 0, 1, 2, 1]
        if pre:
            k = order[0]
            g.prefetch([pinned[2 * k][0], pinned[2 * k + 1][0]], [pinned[2 * k][1], pinned[2 * k + 1][1]])
        for i, k in enumerate(order):
            if pre and i + 1 < len(order) and i != 3:  # step 4 runs without a staged slot
                kn = order[i + 1]
                g.prefetch([pinned[2 * kn][0], pinned[2 * kn + 1][0]], [pinned[2 * kn][1], pinned[2 * kn + 1][1]])
            xs = [pinned[2 * k][0], pinned[2 * k + 1][0]]
            ts = [pinned[2 * k][1], pinned[2 * k + 1][1]]
            losses.append(g.run_step(xs, ts, hp.HyperParams(lr=0.01), device=False).metrics.loss)
            io.append(g.last_step_io()[0])
        res.append((losses, io, [g.param(w, which, l) for w in range(2) for which in range(8)
                                 for l in range(3 if (which & 3) < 2 else 2)]))
    assert res[0][0] == res[1][0]
    assert res[0][1] == res[1][1]
    for a, b in zip(res[0][2], res[1][2]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("math", [hp.MathMode.F32X3, hp.MathMode.BF16])
def test_skip_sync_broadcast_negative_control(math):
    """Cluster::set_skip_sync_broadcast (cluster.cpp:306-314): each worker keeps
    the mean only on its own shard of the flattened conv gradient, so replicas
    diverge exactly as the oracle's do."""
    compare(hp.tiny_cnn(), 4, "B", False, math, 8, skip=True)


@pytest.mark.parametrize("math,K", [(hp.MathMode.F32X3, 2), (hp.MathMode.F32X3, 3), (hp.MathMode.BF16, 2)])
def test_pure_data_parallel_matches_scheme_a(math, K):
    """Scheme DP (BASELINE config 5's pure-data-parallel comparison): each worker
    runs the replicated FC stack on its own examples and the FC gradients are
    all-reduced -- the same exact-SGD update as scheme A on the K*b batch, so
    the oracle's scheme-A run is the reference; every worker's FC copy matches it."""
    spec = hp.tiny_cnn()
    b = 8
    g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=hp.Scheme.DP, seed=1,
                                          math_mode=math))
    o = O.OracleCluster(spec, workers=K, per_worker_batch=b, scheme="A", precision="single", seed=1)
    hpg = hp.HyperParams(momentum=0.9, lr=0.05, weight_decay=5e-4)
    hpo = O.make_hyper_c(0.9, 0.05, 5e-4)
    # (no decision replay here: the oracle's scheme-A fc runs once over the K*b
    # batch, the GPU's replicas once per worker; bf16 keeps the flip-level bound)
    mt, wt, lt = TOL[math] if math != hp.MathMode.BF16 else (3e-1, 5e-4, 1e-4)
    for s in range(2):
        xs, ts = zip(*[hp.synthetic_batch(spec, b, step=s, worker=w) for w in range(K)])
        r = g.run_step(list(xs), list(ts), hpg)
        m = o.run_step([x.astype(np.float64) for x in xs], [t.astype(np.float64) for t in ts], hpo)
        assert abs(r.metrics.loss - m.loss) <= lt * abs(m.loss), (r.metrics.loss, m.loss)
        assert [e.phase for e in r.trace] == [0, 1, 2, 3, 4]
    # gathered_model (cluster.cpp:417-437): worker 0's conv replica and the whole
    # fc matrices, against the oracle's gathered model
    (gconv, gfc), (oconv, ofc) = g.gathered_model(), o.gathered_model()
    for (gk, gb), (ok, ob) in zip(gconv, oconv):
        assert rel_err(gk.ravel(), np.asarray(ok).ravel()) <= wt and rel_err(gb, np.asarray(ob).ravel()) <= mt
    for (gw, gb), (ow, ob) in zip(gfc, ofc):
        assert rel_err(gw.ravel(), np.asarray(ow).ravel()) <= wt and rel_err(gb, np.asarray(ob).ravel()) <= mt
    for w in range(K):
        for l in range(len(spec.conv_layers)):
            for which in (0, 1):
                e = rel_err(g.param(w, which, l), o.param(0, which, l))
                assert e <= (mt if which == 1 else wt), (w, which, l, e)
        for l in range(len(spec.fc_layers)):
            fin = spec.fc_layers[l].in_dim
            full_w = np.concatenate([o.param(k, 2, l).reshape(fin, -1) for k in range(K)], axis=1).ravel()
            full_b = np.concatenate([o.param(k, 3, l) for k in range(K)])
            assert rel_err(g.param(w, 2, l).ravel(), full_w) <= wt, (w, l)
            assert rel_err(g.param(w, 3, l), full_b) <= mt, (w, l)
