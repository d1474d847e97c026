"""Pins the oracle: the C restatement (oracle/hpsim_oracle.c) must be
bit-identical to the unmodified reference (oracle/_ref, compiled from
/root/reference) in double precision — whole run_step (all schemes, K, modes,
counters, trace) and each primitive. Where the reference is not built (the
GPU box), the committed golden fixtures from tests/golden/make_golden.py are
the comparison."""
import os

import numpy as np
import pytest

import oracle as O
from helpers import one_hot, toy_spec

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built (no /root/reference)")


def test_golden_gaussian():
    g = np.load(GOLDEN)
    assert np.array_equal(O.gaussian(0, 64), g["gauss_seed0"])
    assert np.array_equal(O.gaussian(12345, 64), g["gauss_seed12345"])


def test_golden_cluster_steps():
    """Restatement replays the reference's recorded trajectories bit-exactly."""
    g = np.load(GOLDEN)
    spec = toy_spec()
    for ci, (K, s, var, prec) in enumerate(g["cases"]):
        K = int(K)
        c = O.OracleCluster(spec, workers=K, per_worker_batch=4, scheme="ABC"[s], variable_batch=bool(var),
                            precision="single" if prec == 0 else "double", seed=3)
        for w in range(K):
            for which in (0, 2):
                for l in range(2):
                    c.write_param(w, which, l, c.param(w, which, l) * 30.0)
        hp = O.make_hyper_c(0.9, 0.05, 5e-4)
        for st in range(3):
            xs = [g[f"c{ci}_s{st}_x{w}"] for w in range(K)]
            ts = [g[f"c{ci}_s{st}_t{w}"] for w in range(K)]
            m = c.run_step(xs, ts, hp)
            assert list(m.bytes_sent) == list(g[f"c{ci}_s{st}_bytes"])
            assert np.array_equal(np.array(c.trace(), dtype=np.int64), g[f"c{ci}_s{st}_trace"])
            if prec == 1:
                assert m.loss == g[f"c{ci}_loss"][st]
        if prec == 1:  # double: bit-exact; single: the reference rounds every op to float
            for w in range(K):
                for which in range(8):
                    for l in range(2):
                        assert np.array_equal(c.param(w, which, l), g[f"c{ci}_w{w}_p{which}_l{l}"])


@needs_ref
@pytest.mark.parametrize("K", [1, 2, 4])
@pytest.mark.parametrize("scheme,var", [("A", False), ("B", False), ("B", True), ("C", False), ("C", True)])
def test_run_step_bit_exact(K, scheme, var):
    spec = toy_spec()
    kw = dict(workers=K, per_worker_batch=4, scheme=scheme, variable_batch=var, precision="double", seed=1)
    o, r = O.OracleCluster(spec, **kw), O.RefCluster(spec, **kw)
    rng = np.random.default_rng(K * 10 + len(scheme))
    for w in range(K):
        for which in range(4):
            for l in range(2):
                x = rng.normal(size=o.param(w, which, l).size) * 0.3
                o.write_param(w, which, l, x)
                r.write_param(w, which, l, x)
    hp = O.make_hyper_c(0.9, 0.05, 5e-4, fc_partial_lr=0.02 if var else None)
    for _ in range(3):
        xs = [rng.normal(size=(4, 2, 6, 6)) for _ in range(K)]
        ts = [one_hot(rng.integers(0, 4, size=4), 4) for _ in range(K)]
        mo, mr = o.run_step(xs, ts, hp), r.run_step(xs, ts, hp)
        assert mo.loss == mr.loss
        assert list(mo.bytes_sent) == list(mr.bytes_sent)
        assert (mo.fc_update_count, mo.conv_update_count) == (mr.fc_update_count, mr.conv_update_count)
        assert o.trace() == r.trace()
    for w in range(K):
        assert o.worker_bytes(w) == r.worker_bytes(w)
        for which in range(8):
            for l in range(2):
                assert np.array_equal(o.param(w, which, l), r.param(w, which, l))


@needs_ref
def test_skip_sync_broadcast_negative_control():
    spec = toy_spec()
    kw = dict(workers=4, per_worker_batch=4, scheme="B", precision="double", seed=2)
    o, r = O.OracleCluster(spec, **kw), O.RefCluster(spec, **kw)
    o.set_skip_sync_broadcast(True)
    r.set_skip_sync_broadcast(True)
    rng = np.random.default_rng(0)
    xs = [rng.normal(size=(4, 2, 6, 6)) for _ in range(4)]
    ts = [one_hot(rng.integers(0, 4, size=4), 4) for _ in range(4)]
    o.run_step(xs, ts, O.make_hyper_c())
    r.run_step(xs, ts, O.make_hyper_c())
    for w in range(4):
        for l in range(2):
            assert np.array_equal(o.param(w, 0, l), r.param(w, 0, l))
    assert not np.array_equal(o.param(0, 0, 0), o.param(1, 0, 0))


@needs_ref
def test_gaussian_matches_reference():
    lib = O.ref_lib()
    out = np.empty(1000)
    lib.ref_gaussian_fill(77, O._dp(out), 1000)
    assert np.array_equal(out, O.gaussian(77, 1000))


@needs_ref
@pytest.mark.parametrize("stride,pad,floor", [(1, 1, 0), (2, 1, 0), (2, 0, 0), (3, 2, 0)])
def test_conv_primitives(stride, pad, floor):
    rng = np.random.default_rng(stride * 7 + pad)
    B, C, H, W, F, R = 2, 3, 9, 9, 4, 3
    if (H + 2 * pad - R) % stride:
        H = W = H + (stride - (H + 2 * pad - R) % stride)
    x = rng.normal(size=(B, C, H, W)); k = rng.normal(size=(F, C, R, R))
    OH = (H + 2 * pad - R) // stride + 1
    yo = np.empty((B, F, OH, OH)); yr = np.empty_like(yo)
    lib, ref = O.oracle_lib(), O.ref_lib()
    assert lib.or_conv2d_forward(O._dp(x), B, C, H, W, O._dp(k), F, R, R, stride, pad, floor, O._dp(yo)) == 0
    assert ref.ref_conv2d_forward(1, O._dp(x), B, C, H, W, O._dp(k), F, R, R, stride, pad, O._dp(yr)) == 0
    assert np.array_equal(yo, yr)
    gy = rng.normal(size=yo.shape)
    gxo, gko = np.empty_like(x), np.empty_like(k)
    gxr, gkr = np.empty_like(x), np.empty_like(k)
    lib.or_conv2d_backward(O._dp(x), B, C, H, W, O._dp(k), F, R, R, stride, pad, floor, O._dp(gy), O._dp(gxo), O._dp(gko))
    ref.ref_conv2d_backward(1, O._dp(x), B, C, H, W, O._dp(k), F, R, R, stride, pad, O._dp(gy), OH, OH,
                            O._dp(gxr), O._dp(gkr))
    assert np.array_equal(gxo, gxr) and np.array_equal(gko, gkr)


@needs_ref
def test_matmul_xent_momentum_primitives():
    rng = np.random.default_rng(3)
    lib, ref = O.oracle_lib(), O.ref_lib()
    a = rng.normal(size=(5, 7)); b = rng.normal(size=(7, 3))
    co, cr = np.empty((5, 3)), np.empty((5, 3))
    lib.or_matmul(O._dp(a), O._dp(b), O._dp(co), 5, 7, 3)
    ref.ref_matmul(1, 0, O._dp(a), O._dp(b), O._dp(cr), 5, 7, 7, 3)
    assert np.array_equal(co, cr)
    at = rng.normal(size=(7, 5))
    lib.or_matmul_tn(O._dp(at), O._dp(b), O._dp(co), 7, 5, 3)
    ref.ref_matmul(1, 1, O._dp(at), O._dp(b), O._dp(cr), 7, 5, 7, 3)
    assert np.array_equal(co, cr)
    bn = rng.normal(size=(3, 7))
    lib.or_matmul_nt(O._dp(a), O._dp(bn), O._dp(co), 5, 7, 3)
    ref.ref_matmul(1, 2, O._dp(a), O._dp(bn), O._dp(cr), 5, 7, 3, 7)
    assert np.array_equal(co, cr)
    z = rng.normal(size=(4, 6)) * 5; t = rng.uniform(size=(4, 6))
    go, gr = np.empty_like(z), np.empty_like(z)
    lo, lr = np.zeros(1), np.zeros(1)
    lib.or_logistic_xent(O._dp(z), O._dp(t), 4, 6, O._dp(go), O._dp(lo))
    ref.ref_logistic_xent(1, O._dp(z), O._dp(t), 4, 6, O._dp(gr), O._dp(lr))
    assert lo[0] == lr[0] and np.array_equal(go, gr)
    w = rng.normal(size=50); d = rng.normal(size=50); g = rng.normal(size=50)
    w2, d2 = w.copy(), d.copy()
    lib.or_momentum_update(O._dp(w), O._dp(d), O._dp(g), 50, 0.01, 0.9, 5e-4)
    ref.ref_momentum_update(1, O._dp(w2), O._dp(d2), O._dp(g), 50, 0.01, 0.9, 5e-4)
    assert np.array_equal(w, w2) and np.array_equal(d, d2)
    # float storage (what the GPU SGD kernel must equal bit-for-bit)
    wf, df, gf = (v.astype(np.float32) for v in (w, d, g))
    wr, dr = wf.astype(np.float64), df.astype(np.float64)
    F = O.C.POINTER(O.C.c_float)
    lib.or_momentum_update_f32(wf.ctypes.data_as(F), df.ctypes.data_as(F), gf.ctypes.data_as(F), 50, 0.01, 0.9, 5e-4)
    ref.ref_momentum_update(0, O._dp(wr), O._dp(dr), O._dp(gf.astype(np.float64)), 50, 0.01, 0.9, 5e-4)
    assert np.array_equal(wf.astype(np.float64), wr) and np.array_equal(df.astype(np.float64), dr)


@needs_ref
def test_validation_messages_match_reference():
    """ConfigError paths: same code (and the reference's field-path message)."""
    spec = toy_spec()
    bad = toy_spec()
    bad.conv_layers[1].in_channels = 5
    for s, kw in [(bad, {}), (spec, dict(workers=3, per_worker_batch=128, scheme="C")),
                  (spec, dict(workers=2, per_worker_batch=4, scheme="A", variable_batch=True))]:
        with pytest.raises(O.OracleError) as eo:
            O.OracleCluster(s, **kw)
        with pytest.raises(O.OracleError) as er:
            O.RefCluster(s, **kw)
        assert eo.value.code == er.value.code == 1
        assert str(eo.value) == str(er.value)
