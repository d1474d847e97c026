"""The C restatement (oracle/) against SPEC.md's known-answer tests and
acceptance properties. CPU only."""
import math

import numpy as np
import pytest

import oracle as O
from helpers import one_hot, rel_err, toy_spec


def test_xent_kats():
    lib = O.oracle_lib()
    z = np.array([0.0]); t = np.array([1.0]); g = np.zeros(1); loss = np.zeros(1)
    assert lib.or_logistic_xent(O._dp(z), O._dp(t), 1, 1, O._dp(g), O._dp(loss)) == 0
    assert abs(loss[0] - math.log(2)) < 1e-15 and g[0] == -0.5
    z = np.array([40.0])
    lib.or_logistic_xent(O._dp(z), O._dp(t), 1, 1, O._dp(g), O._dp(loss))
    assert loss[0] < 1e-15 and abs(g[0]) < 1e-15
    t = np.array([1.5])
    assert lib.or_logistic_xent(O._dp(z), O._dp(t), 1, 1, O._dp(g), O._dp(loss)) == 3  # DomainError


def test_momentum_kats():
    lib = O.oracle_lib()
    w = np.zeros(1); d = np.zeros(1); g = np.ones(1)
    lib.or_momentum_update(O._dp(w), O._dp(d), O._dp(g), 1, 0.1, 0.0, 0.0)
    assert w[0] == pytest.approx(-0.1) and d[0] == pytest.approx(-0.1)
    w = np.zeros(1); d = np.zeros(1)
    for _ in range(2):
        lib.or_momentum_update(O._dp(w), O._dp(d), O._dp(g), 1, 0.1, 0.9, 0.0)
    assert d[0] == pytest.approx(-0.19, abs=1e-15) and w[0] == pytest.approx(-0.29, abs=1e-15)
    w = np.array([2.0]); d = np.zeros(1); g = np.zeros(1)
    lib.or_momentum_update(O._dp(w), O._dp(d), O._dp(g), 1, 0.1, 0.0, 0.5)
    assert w[0] == pytest.approx(2.0 * (1 - 0.1 * 0.5))


def _run(K, scheme, var, steps, b=4, lr=0.05, mu=0.9, wd=5e-4, seed=3, data_seed=11, scale=30.0):
    spec = toy_spec()
    c = O.OracleCluster(spec, workers=K, per_worker_batch=b, scheme=scheme, variable_batch=var, seed=seed)
    for w in range(K):
        for which in (0, 2):
            for l in range(2):
                c.write_param(w, which, l, c.param(w, which, l) * scale)
    rng = np.random.default_rng(data_seed)
    hp = O.make_hyper_c(mu, lr, wd)
    ms = []
    for _ in range(steps):
        xs = [rng.normal(size=(b, 2, 6, 6)) for _ in range(K)]
        ts = [one_hot(rng.integers(0, 4, size=b), 4) for _ in range(K)]
        ms.append(c.run_step(xs, ts, hp))
    return c, ms


@pytest.mark.parametrize("K", [1, 2, 4])
@pytest.mark.parametrize("scheme", ["A", "B", "C"])
def test_synchronous_equivalence(K, scheme):
    """Acceptance 1: K workers == single-model SGD at batch K*b, 5 steps, < 1e-8."""
    c, _ = _run(K, scheme, False, 5)
    # single worker at batch K*b on the same data (concatenate the K batches)
    spec = toy_spec()
    s = O.OracleCluster(spec, workers=1, per_worker_batch=4 * K, scheme="B", seed=3)
    for which in (0, 2):
        for l in range(2):
            s.write_param(0, which, l, s.param(0, which, l) * 30.0)
    rng = np.random.default_rng(11)
    hp = O.make_hyper_c(0.9, 0.05, 5e-4)
    for _ in range(5):
        xs = [rng.normal(size=(4, 2, 6, 6)) for _ in range(K)]
        ts = [one_hot(rng.integers(0, 4, size=4), 4) for _ in range(K)]
        s.run_step([np.concatenate(xs)], [np.concatenate(ts)], hp)
    cm, fm = c.gathered_model()
    sm, sf = s.gathered_model()
    worst = max(max(rel_err(a, b) for a, b in zip(x, y)) for x, y in zip(cm + fm, sm + sf))
    assert worst < 1e-8
    # replica consistency: conv params bit-identical across workers
    for w in range(1, K):
        for l in range(2):
            assert np.array_equal(c.param(w, 0, l), c.param(0, 0, l))


@pytest.mark.parametrize("K", [2, 4, 8])
def test_pass_counts_and_bottleneck(K):
    """Acceptance 5/6: passes 2+2K (B/C) and 4 (A); max-sender bytes B=(K-1)b*A_bytes, C=(K-1)/K*b*A_bytes."""
    b, A_bytes = 16, 36 * 8
    for scheme, passes in (("A", 4), ("B", 2 + 2 * K), ("C", 2 + 2 * K)):
        c, _ = _run(K, scheme, False, 1, b=b)
        tr = c.trace()
        assert sum(1 for e in tr if e[0] != 4) == passes
        fwd = [e for e in tr if e[0] == 1]
        if scheme == "B":
            assert all(e[4] == (K - 1) * b * A_bytes for e in fwd)
        if scheme == "C":
            assert all(e[4] == (K - 1) * (b // K) * A_bytes for e in fwd)


def test_sync_bytes_uneven():
    """Sync bytes per worker (G-s_i)e + (K-1)s_i e with the last shard taking the
    remainder (cluster.cpp:297-304; G=109, K=4 -> 1304 B in double)."""
    _, _ = _run(4, "B", False, 1)
    G = 3 * 2 * 9 + 3 + 4 * 3 * 4 + 4  # toy conv params = 109
    assert G == 109
    c, _ = _run(4, "B", False, 1)
    for i in range(4):
        s, r = c.worker_bytes(i)
        s0, s1 = (27 * i, 27 * (i + 1)) if i < 3 else (81, 109)
        assert s[3] == ((G - (s1 - s0)) + 3 * (s1 - s0)) * 8
    assert c.worker_bytes(0)[0][3] == 1304


def test_variable_lr0_equals_uniform():
    """Acceptance 10: variable mode with eps=0 == uniform mode bit-exactly; K FC updates/step."""
    for scheme in ("B", "C"):
        a, ma = _run(4, scheme, True, 3, lr=0.0)
        u, mu_ = _run(4, scheme, False, 3, lr=0.0)
        assert all(m.fc_update_count == 4 for m in ma) and all(m.fc_update_count == 1 for m in mu_)
        for w in range(4):
            for which in range(8):
                for l in range(2):
                    assert np.array_equal(a.param(w, which, l), u.param(w, which, l))


def test_finite_differences():
    """Acceptance 9: end-to-end gradient vs central differences (double), < 1e-5.
    Gradient via one step with mu=wd=0, lr=1 (w' = w - g); loss via lr=0 steps."""
    spec = toy_spec()
    rng = np.random.default_rng(5)
    x = rng.normal(size=(3, 2, 6, 6)); t = one_hot(rng.integers(0, 4, size=3), 4)

    def fresh():
        c = O.OracleCluster(spec, workers=1, per_worker_batch=3, scheme="B", seed=9)
        for which in (0, 2):
            for l in range(2):
                c.write_param(0, which, l, c.param(0, which, l) * 30.0)
        return c
    base = fresh()
    params = {(w, l): base.param(0, w, l) for w in range(4) for l in range(2)}
    g = fresh()
    g.run_step([x], [t], O.make_hyper_c(0.0, 1.0, 0.0))
    worst = 0.0
    for _ in range(20):
        which, l = int(rng.integers(0, 4)), int(rng.integers(0, 2))
        p = params[(which, l)]
        k = int(rng.integers(0, p.size))
        grad = p[k] - g.param(0, which, l)[k]
        h = 1e-5
        vals = []
        for sgn in (1, -1):
            c = fresh()
            q = p.copy(); q[k] += sgn * h
            c.write_param(0, which, l, q)
            vals.append(c.run_step([x], [t], O.make_hyper_c(0.0, 0.0, 0.0), lr=0.0).loss)
        fd = (vals[0] - vals[1]) / (2 * h)
        if abs(fd) > 1e-7:
            worst = max(worst, abs(fd - grad) / abs(fd))
    assert worst < 1e-5


def test_config_guards():
    spec = toy_spec()
    with pytest.raises(O.OracleError) as e:
        O.OracleCluster(spec, workers=3, per_worker_batch=128, scheme="C")
    assert e.value.code == 1 and "not divisible by 3" in str(e.value)
    with pytest.raises(O.OracleError) as e:
        O.OracleCluster(spec, workers=2, per_worker_batch=4, scheme="A", variable_batch=True)
    assert e.value.code == 1
