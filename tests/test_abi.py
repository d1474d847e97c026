"""C ABI boundary (CPU): the library loads, exports every entry point the
header declares, and the host-side logic (validation with the reference's
error types and messages, shard_range, GaussianSampler replay) matches the
reference / oracle. No GPU compute is called here."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
import paper_1404_5997_b200 as hp
from paper_1404_5997_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "hpsim_b200.h")).read()
    return sorted(set(re.findall(r"HP_API\s+[\w\s\*]+?\b(hp_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    syms = header_symbols()
    assert len(syms) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (hp_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    for s in syms:
        assert getattr(_lib.lib, s) is not None


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_shard_range_matches_reference_rule():
    for total, parts in [(10, 4), (4096, 8), (1000, 8), (256, 3), (7, 7)]:
        for i in range(parts):
            b, e = hp.shard_range(total, parts, i)
            base = total // parts
            assert b == base * i and e == (total if i == parts - 1 else b + base)


def test_gaussian_replay_matches_oracle():
    assert np.array_equal(hp.gaussian(123, 1001), O.gaussian(123, 1001))
    assert np.array_equal(hp.gaussian_f32(5, 100, 0.01), (0.01 * O.gaussian(5, 100)).astype(np.float32))


def test_mt19937_64_labels():
    from paper_1404_5997_b200.specs import mt19937_64
    assert np.array_equal(mt19937_64(42, 700), O.uniform_u64(42, 700))
    assert int(mt19937_64(5489, 1)[0]) == 14514284786278117030  # std::mt19937_64 default-seed KAT


@pytest.mark.parametrize("mutate,needle", [
    (lambda s, c: setattr(c, "scheme", hp.Scheme.C) or setattr(c, "workers", 3), "not divisible by 3"),
    (lambda s, c: setattr(c, "scheme", hp.Scheme.A) or setattr(c, "variable_batch", True) or setattr(c, "workers", 2),
     "scheme A has a single fc pass"),
    (lambda s, c: setattr(c, "precision", hp.Precision.DOUBLE), "cluster.precision"),
    (lambda s, c: setattr(c, "workers", 0), "cluster.workers: must be >= 1"),
    (lambda s, c: setattr(s.conv_layers[1], "in_channels", 7), "model.conv_layers[1].in_channels: expected 32, got 7"),
    (lambda s, c: setattr(s.fc_layers[0], "in_dim", 100), "model.fc_layers[0].in_dim: expected 4096"),
    (lambda s, c: setattr(s, "num_classes", 11), "does not match num_classes"),
    (lambda s, c: setattr(s.conv_layers[0], "kernel", 4), "is not a positive integer"),
    (lambda s, c: setattr(s.conv_layers[0], "out_channels", 30) or setattr(s.conv_layers[1], "in_channels", 30),
     "multiple of 8"),
])
def test_config_errors(mutate, needle):
    spec = hp.tiny_cnn()
    cfg = hp.ClusterConfig(workers=1, per_worker_batch=128)
    mutate(spec, cfg)
    with pytest.raises(hp.ConfigError) as e:
        hp.Cluster(spec, cfg)
    assert needle in str(e.value)


def test_reference_rejects_alexnet_224_and_we_accept_floor_mode():
    spec = hp.alexnet_1col()
    assert spec.flattened_conv_size() == 9216
    spec.conv_layers[0].floor_mode = False
    with pytest.raises(hp.ConfigError) as e:
        hp.Cluster(spec, hp.ClusterConfig())
    assert "(224+2*2-11)/4+1 is not a positive integer" in str(e.value)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1404_5997_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".hpp", "Makefile")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "hpsim_oracle" not in txt and "libhpsim_ref" not in txt, f


def test_pure_dp_accounting():
    """Scheme DP (B200 extension, BASELINE config 5): no boundary / FC-internal
    traffic; the conv and FC gradient vectors are each all-reduced and charged
    with the reference's sync formula (G - s_i)*4 + (K-1)*s_i*4 (cluster.cpp:296-304)."""
    spec = hp.alexnet_1col()
    K = 8
    bs, trace, per = hp.step_accounting(spec, hp.ClusterConfig(workers=K, per_worker_batch=128,
                                                               scheme=hp.Scheme.DP))
    Gc = sum(l.out_channels * l.in_channels * l.kernel ** 2 + l.out_channels for l in spec.conv_layers)
    Gf = sum(f.in_dim * f.out_dim + f.out_dim for f in spec.fc_layers)
    assert Gc == 3_207_104 and Gc + Gf == 61_838_248

    def charge(G, i):
        s0, s1 = hp.shard_range(G, K, i)
        return (G - (s1 - s0)) * 4 + (K - 1) * (s1 - s0) * 4
    assert bs[0] == 0 and bs[2] == 0  # fc activations / fc internal (MsgClass order, cluster.hpp)
    assert bs[1] == sum(charge(Gf, i) for i in range(K))
    assert bs[3] == sum(charge(Gc, i) for i in range(K))
    assert [e[0] for e in trace] == [0, 1, 2, 3, 4]
    assert trace[-1][3] == bs[1] + bs[3]
    for i, (sent, recv) in enumerate(per):
        assert sent == [0, charge(Gf, i), 0, charge(Gc, i)] and recv == sent
