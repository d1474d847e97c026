"""SPEC cost_model: footnote KATs, the (K-1)/K hiding law,
bottleneck byte counts against the library's own accounting trace,
monotonicity, the K=8 sanity envelope, and the cost-report CLI (acceptance
criteria 2-4). (hparam_scaling is out of scope: SURVEY §2.1.)"""
import dataclasses
import json
import math
import random

import pytest

from paper_1404_5997_b200 import api as hp, cli
from paper_1404_5997_b200 import cost_model as cm
from paper_1404_5997_b200.specs import alexnet_1col, tiny_cnn


def fc_heavy_spec():
    """Toy spec whose FC compute per sub-batch dwarfs the boundary broadcast."""
    return hp.ModelSpec(conv_layers=[hp.ConvLayerSpec(3, 8, 4, 4, 0)],
                        fc_layers=[hp.FcLayerSpec(512, 4096, True), hp.FcLayerSpec(4096, 4096, True),
                                   hp.FcLayerSpec(4096, 10, False)],
                        input_shape=[3, 32, 32], num_classes=10)


# ---------------------------------------------------------------- footnote arithmetic (criterion 3)
def test_footnote_arithmetic():
    assert 2.09e-6 <= cm.compute_time(4096 * 512 * 2, cm.PAPER) <= 2.10e-6
    assert cm.compute_time(0, cm.PAPER) == 0 and cm.compute_time(2e12, cm.PAPER) == 1.0
    assert 2.73e-6 <= cm.comm_time(16384, cm.PAPER) <= 2.74e-6
    assert cm.comm_time(0, cm.PAPER) == 0
    p0 = dataclasses.replace(cm.PAPER, host_hop_latency=0.0)
    assert cm.comm_time(16384, p0, same_subset=False) == pytest.approx(5.4613e-6, rel=1e-4)
    assert cm.comm_time(0, cm.PAPER, same_subset=False) == cm.PAPER.host_hop_latency
    assert cm.comm_time(16384, cm.PAPER, concurrent_flows=4) == pytest.approx(4 * 16384 / 6e9)
    b = cm.fc_matmul_balance(4096, cm.PAPER, K=8)
    assert b["comm_bound"] and b["compute_s"] == pytest.approx(2.097e-6, rel=1e-3)
    b2 = cm.fc_matmul_balance(8192, cm.PAPER, K=8)
    assert not b2["comm_bound"] and b2["compute_s"] == pytest.approx(8.389e-6, rel=1e-3)
    assert b2["comm_s"] == pytest.approx(5.461e-6, rel=1e-3)
    assert cm.fc_matmul_balance(1, cm.PAPER)["comm_bound"]


def test_param_validation():
    with pytest.raises(ValueError):
        cm.CostParams(cross_subset_penalty=0.0)
    with pytest.raises(ValueError):
        cm.CostParams(link_bandwidth=-1)
    with pytest.raises(ValueError):
        cm.Topology(4, [[0, 1], [1, 2, 3]])
    with pytest.raises(ValueError):
        cm.compute_time(-1, cm.PAPER)


# ---------------------------------------------------------------- hiding law (criterion 4)
@pytest.mark.parametrize("K", [2, 4, 8])
def test_scheme_b_hides_k_minus_1_over_k(K):
    spec = fc_heavy_spec()
    cl = hp.ClusterConfig(workers=K, per_worker_batch=32, scheme=hp.Scheme.B)
    for params, topo in ((cm.PAPER, cm.paper_topology(K)), (cm.b200_params(), cm.b200_topology(K))):
        tl = cm.scheme_step_model(spec, cl, topo, params)
        assert tl.hidden_comm_fraction == pytest.approx((K - 1) / K, abs=1e-12)


def test_k1_and_scheme_a():
    spec = alexnet_1col()
    r = cm.speedup(spec, hp.ClusterConfig(workers=1, per_worker_batch=128), cm.Topology(1), cm.PAPER)
    assert r["speedup"] == 1.0 and r["hidden_comm_fraction"] is None
    tl = cm.scheme_step_model(spec, hp.ClusterConfig(workers=4, per_worker_batch=128, scheme=hp.Scheme.A),
                              cm.paper_topology(4), cm.PAPER)
    assert tl.hidden_comm_fraction == 0.0  # scheme (a): "all useful work has to pause"


# ---------------------------------------------------------------- bottleneck bytes (criterion 5)
@pytest.mark.parametrize("K", [2, 4, 8])
def test_bottleneck_bytes_match_accounting(K):
    spec, b = tiny_cnn(), 16
    A = spec.flattened_conv_size()
    got = {}
    for s in (hp.Scheme.A, hp.Scheme.B, hp.Scheme.C):
        x = cm.exchange_elements(spec, K, b, s)
        _, trace, _ = hp.step_accounting(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=s))
        fwd = [e for e in trace if e[0] == hp.Phase.FC_FWD]
        bwd = [e for e in trace if e[0] == hp.Phase.FC_BWD]
        assert len(fwd) == x["turns"] == len(bwd)
        assert all(e[4] == x["act"] * 4 for e in fwd)   # f32 wire elements
        assert all(e[4] == x["grad"] * 4 for e in bwd)
        got[s] = x["act"]
    assert got[hp.Scheme.B] == (K - 1) * b * A
    assert got[hp.Scheme.C] == (K - 1) * (b // K) * A < b * A
    assert got[hp.Scheme.C] / got[hp.Scheme.B] == pytest.approx(1 / K)


# ---------------------------------------------------------------- timeline properties
@pytest.mark.parametrize("scheme", [hp.Scheme.A, hp.Scheme.B, hp.Scheme.C, hp.Scheme.DP])
def test_timeline_conservation_and_no_compute_overlap(scheme):
    spec, K, b = alexnet_1col(), 4, 64
    tl = cm.scheme_step_model(spec, hp.ClusterConfig(workers=K, per_worker_batch=b, scheme=scheme),
                              cm.paper_topology(K), cm.PAPER)
    comp = sorted((e.t0, e.t1) for e in tl.events if e.kind == "compute")
    for (a0, a1), (b0, b1) in zip(comp, comp[1:]):
        assert a1 <= b0 + 1e-15
    fl = cm.model_flops(spec)
    conv = (3 * sum(fl["conv_fwd"]) - fl["conv_fwd"][0]) * b
    fc = 3 * sum(fl["fc_fwd"]) * (b if scheme == hp.Scheme.DP else b * K / K)
    assert sum(t1 - t0 for t0, t1 in comp) == pytest.approx(cm.compute_time(conv + fc, cm.PAPER), rel=1e-12)
    assert tl.step_time >= max(e.t1 for e in tl.events if e.kind == "compute")


def test_monotone_in_bandwidth_and_flops():
    spec = alexnet_1col()
    for s in (hp.Scheme.A, hp.Scheme.B, hp.Scheme.C, hp.Scheme.DP):
        cl = hp.ClusterConfig(workers=8, per_worker_batch=128, scheme=s)
        prev = None
        for bw in (3e9, 6e9, 12e9, 1e11):
            t = cm.scheme_step_model(spec, cl, cm.paper_topology(8), dataclasses.replace(cm.PAPER, link_bandwidth=bw))
            assert prev is None or t.step_time <= prev
            prev = t.step_time
        prev = None
        for f in (1e12, 2e12, 4e12):
            t = cm.scheme_step_model(spec, cl, cm.paper_topology(8), dataclasses.replace(cm.PAPER, flops_per_sec=f))
            assert prev is None or t.step_time <= prev
            prev = t.step_time


def test_paper_envelope_k8():
    """modeled K=8 speedup with §5's machine in [4, 8]."""
    spec = alexnet_1col()
    for s in (hp.Scheme.A, hp.Scheme.B, hp.Scheme.C):
        r = cm.speedup(spec, hp.ClusterConfig(workers=8, per_worker_batch=128, scheme=s), cm.paper_topology(8),
                       cm.PAPER)
        assert 4.0 <= r["speedup"] <= 8.0


def test_calibration_reproduces_measured_k1():
    spec = alexnet_1col()
    p = cm.b200_params()
    scale = cm.calibrate(spec, 128, p, 1.737e-3)
    t = cm.scheme_step_model(spec, hp.ClusterConfig(workers=1, per_worker_batch=128), cm.Topology(1), p,
                             compute_scale=scale)
    assert t.step_time == pytest.approx(1.737e-3, rel=1e-12)


# ---------------------------------------------------------------- hparam scaling (criterion 2)
def _cfg(tmp_path, **cluster):
    c = {"model": "tiny_cnn", "cluster": dict({"workers": 1, "per_worker_batch": 16, "scheme": "B"}, **cluster),
         "output_dir": str(tmp_path / "out"), "cost": {"machine": "paper"}}
    p = tmp_path / "c.json"
    p.write_text(json.dumps(c))
    return str(p)


def test_cli_cost_report(tmp_path, capsys):
    assert cli.main(["cost-report", "--config", _cfg(tmp_path), "--json"]) == 0
    r = json.loads(capsys.readouterr().out)
    assert r["speedup"] == 1.0 and r["hidden_comm_fraction"] is None
    assert cli.main(["cost-report", "--config", _cfg(tmp_path, workers=4, per_worker_batch=16)]) == 0
    out = capsys.readouterr().out
    assert "hidden_comm_fraction=" in out and "conv_fwd" in out
    rows = (tmp_path / "out" / "timeline.csv").read_text().splitlines()
    assert rows[0] == "worker,t0,t1,kind,label" and len(rows) > 5


def test_cli_cost_report_fc_heavy(tmp_path, capsys):
    spec = fc_heavy_spec()
    c = {"model": {"conv_layers": [dataclasses.asdict(l) for l in spec.conv_layers],
                   "fc_layers": [dataclasses.asdict(f) for f in spec.fc_layers],
                   "input_shape": spec.input_shape, "num_classes": spec.num_classes},
         "cluster": {"workers": 4, "per_worker_batch": 32, "scheme": "B"},
         "output_dir": str(tmp_path / "o"), "cost": {"machine": "paper"}}
    p = tmp_path / "c.json"
    p.write_text(json.dumps(c))
    assert cli.main(["cost-report", "--config", str(p), "--json"]) == 0
    assert json.loads(capsys.readouterr().out)["hidden_comm_fraction"] == pytest.approx(0.75, abs=1e-12)


def test_cli_cost_report_bad_machine(tmp_path):
    p = tmp_path / "c.json"
    p.write_text(json.dumps({"cost": {"machine": "tpu"}, "output_dir": str(tmp_path)}))
    assert cli.main(["cost-report", "--config", str(p)]) == cli.EXIT_VALIDATION


def test_fc_hbm_term_shards_with_model_parallelism():
    """B200 parameter set: FC passes are max(FLOPs, bf16 weight reads) and the
    fused update streams 18 B per parameter a worker holds (1/K shard under
    the hybrid schemes, all of it under pure DP)."""
    spec = alexnet_1col()
    p = cm.b200_params()
    P = sum(f.in_dim * f.out_dim for f in spec.fc_layers)
    t1 = cm.scheme_step_model(spec, hp.ClusterConfig(workers=1, per_worker_batch=128), cm.Topology(1), p)
    assert t1.phase_table()["fc_update"] == pytest.approx(18 * P / p.hbm_bandwidth)
    assert t1.phase_table()["fc"] >= 4 * P / p.hbm_bandwidth
    for s, share in ((hp.Scheme.A, 1 / 8), (hp.Scheme.B, 1 / 8), (hp.Scheme.DP, 1.0)):
        tk = cm.scheme_step_model(spec, hp.ClusterConfig(workers=8, per_worker_batch=128, scheme=s),
                                  cm.b200_topology(8), p)
        assert tk.phase_table()["fc_update"] == pytest.approx(18 * P * share / p.hbm_bandwidth)
    # the paper machine keeps the SPEC's FLOPs-only FC phase
    assert "fc_update" not in cm.scheme_step_model(spec, hp.ClusterConfig(workers=1, per_worker_batch=128),
                                                   cm.Topology(1), cm.PAPER).phase_table()


def test_cli_cost_report_b200_calibrated(tmp_path, capsys):
    """machine b200 + measured_step_ms: the K=1 model reproduces the measured
    step, and the report carries the FC update phase (HBM term)."""
    c = {"model": "alexnet_1col", "cluster": {"workers": 1, "per_worker_batch": 128, "scheme": "B"},
         "output_dir": str(tmp_path / "o"), "cost": {"machine": "b200", "measured_step_ms": 1.6}}
    p = tmp_path / "c.json"
    p.write_text(json.dumps(c))
    assert cli.main(["cost-report", "--config", str(p), "--json"]) == 0
    r = json.loads(capsys.readouterr().out)
    assert r["step_time_K"] == pytest.approx(1.6e-3, rel=1e-9)
    assert "fc_update" in r["phases_s"] and r["speedup"] == pytest.approx(1.0)
    c["cluster"].update(workers=8, scheme="A")
    p.write_text(json.dumps(c))
    assert cli.main(["cost-report", "--config", str(p), "--json"]) == 0
    r8 = json.loads(capsys.readouterr().out)
    assert r8["phases_s"]["fc_update"] == pytest.approx(r["phases_s"]["fc_update"] / 8, rel=1e-9)
