"""SPEC cli_harness on the B200 path: config validation,
metrics CSV schema, checkpoint format, verify-equivalence exit codes."""
import csv
import json
import os

import numpy as np
import pytest

from paper_1404_5997_b200 import cli


def write_cfg(tmp_path, **over):
    cfg = {"model": "tiny_cnn", "cluster": {"workers": 2, "per_worker_batch": 8, "scheme": "B", "seed": 1,
                                            "math_mode": "bf16"},
           "hyper": {"lr": 0.01}, "steps": 3, "output_dir": str(tmp_path / "out")}
    for k, v in over.items():
        if isinstance(v, dict) and isinstance(cfg.get(k), dict):
            cfg[k].update(v)
        else:
            cfg[k] = v
    p = tmp_path / "run.json"
    p.write_text(json.dumps(cfg))
    return str(p)


def test_config_round_trip_and_defaults(tmp_path):
    cfg = cli.load_config(write_cfg(tmp_path))
    again = cli.normalize_config(json.loads(json.dumps(cfg)))
    assert again == cfg  # load -> serialize -> load is identity
    assert cfg["hyper"]["momentum"] == 0.9 and cfg["data"]["seed_data"] == 100


@pytest.mark.parametrize("over,msg", [
    ({"cluster": {"scheme": "X"}}, "config.cluster.scheme"),
    ({"cluster": {"workers": 0}}, "config.cluster.workers"),
    ({"bogus": 1}, "unknown field"),
    ({"model": "vgg"}, "config.model"),
    ({"cluster": {"scheme": "C", "workers": 3}}, "per_worker_batch"),  # K | b for scheme C (library check)
])
def test_validation_exit_code_1(tmp_path, capsys, over, msg):
    rc = cli.main(["train", "--config", write_cfg(tmp_path, **over)])
    assert rc == cli.EXIT_VALIDATION
    assert msg in capsys.readouterr().err


@pytest.mark.parametrize("data,msg", [
    ({"generator": "gaussian_blobs", "num_examples": 20}, "multiple of K*b"),
    ({"generator": "mnist", "num_examples": 32}, "gaussian_blobs"),
])
def test_data_generator_validation(tmp_path, capsys, data, msg):
    rc = cli.main(["train", "--config", write_cfg(tmp_path, data=data)])
    assert rc == cli.EXIT_VALIDATION
    assert msg in capsys.readouterr().err


@pytest.mark.gpu
def test_train_on_generated_device_batches(tmp_path):
    """SPEC data_gen as the input pipeline: batches generated on the GPU into the
    step's device inputs; epochs partition the dataset (epoch column advances)."""
    rc = cli.main(["train", "--config", write_cfg(tmp_path, steps=6, data={
        "generator": "gaussian_blobs", "num_examples": 32, "seed": 3, "separation": 0.5})])
    assert rc == 0
    rows = list(csv.reader(open(tmp_path / "out" / "metrics.csv")))[1:]
    assert [int(r[1]) for r in rows] == [0, 0, 1, 1, 2, 2]
    assert all(np.isfinite(float(r[2])) for r in rows)


def test_zero_steps_header_only_csv(tmp_path):
    rc = cli.main(["train", "--config", write_cfg(tmp_path, steps=0)])
    assert rc == 0
    rows = list(csv.reader(open(tmp_path / "out" / "metrics.csv")))
    assert rows == [cli.CSV_HEADER]
    assert ",".join(cli.CSV_HEADER) == ("step,epoch,loss,lr,bytes_fc_activations,bytes_fc_gradients,"
                                        "bytes_fc_internal,bytes_conv_sync,sim_step_time_s,wall_time_s")


def test_checkpoint_raw_le_float32_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    ts = [("conv0.kernels", [4, 3, 2, 2], rng.standard_normal(48).astype(np.float32)),
          ("fc0.bias", [5], rng.standard_normal(5).astype(np.float32))]
    cli.write_checkpoint(str(tmp_path / "ck"), ts)
    man = json.load(open(tmp_path / "ck" / "manifest.json"))
    assert [t["name"] for t in man["tensors"]] == ["conv0.kernels", "fc0.bias"]
    assert os.path.getsize(tmp_path / "ck" / "conv0.kernels.f32") == 48 * 4
    back = cli.read_checkpoint(str(tmp_path / "ck"))
    assert np.array_equal(back["conv0.kernels"].ravel(), ts[0][2]) and back["fc0.bias"].dtype == np.dtype("<f4")


@pytest.mark.gpu
def test_train_metrics_checkpoint_and_determinism(tmp_path):
    import paper_1404_5997_b200 as hp
    rows = []
    for run in range(2):
        out = tmp_path / f"o{run}"
        assert cli.main(["train", "--config", write_cfg(tmp_path, output_dir=str(out))]) == 0
        r = list(csv.reader(open(out / "metrics.csv")))
        assert r[0] == cli.CSV_HEADER and len(r) == 4
        rows.append([row[:-1] for row in r[1:]])  # all but wall_time
        ck = cli.read_checkpoint(str(out / "checkpoint"))
        assert set(ck) == {f"conv{l}.{k}" for l in range(3) for k in ("kernels", "bias")} | \
            {f"fc{l}.{k}" for l in range(2) for k in ("weight", "bias")}
    assert rows[0] == rows[1]  # deterministic per config + seed
    assert float(rows[0][0][2]) > 0 and int(rows[0][0][4]) > 0  # loss, fc activation bytes (K=2 scheme B)


@pytest.mark.gpu
def test_verify_equivalence_and_negative_control(tmp_path, capsys):
    path = write_cfg(tmp_path, steps=2)
    assert cli.main(["verify-equivalence", "--config", path]) == 0
    out = capsys.readouterr().out
    assert "scheme A" in out and "scheme B" in out and "scheme C" in out
    assert cli.main(["verify-equivalence", "--config", path, "--skip-broadcast"]) == cli.EXIT_EQUIVALENCE
