"""Command-line harness on the B200 path (SPEC.md `cli_harness`, 522-583): the
step either side of `Cluster::run_step` that makes B200 runs diffable.

  python -m paper_1404_5997_b200.cli train --config run.json
      runs `steps` steps on synthetic data, writes <output_dir>/metrics.csv
      (header exactly SPEC.md:569) and <output_dir>/checkpoint/ (one raw
      little-endian float32 file per parameter tensor of the gathered model +
      manifest.json with names / shapes / precision).
  python -m paper_1404_5997_b200.cli verify-equivalence --config run.json
      §4.2 "completely equivalent to synchronous SGD on the K*b batch": runs the
      config's K workers under schemes A, B, C (exact, 3xTF32 parity math) and a
      single worker on the concatenated K*b batch, all on the B200 path, prints
      the max relative parameter divergence per scheme; exit 0 iff all are
      within `--tol` (the 3xTF32 tolerance), 3 otherwise.
      `--skip-broadcast` is the negative control (cluster.hpp:203-205).

Exit codes: 0 success, 1 validation, 2 runtime, 3 equivalence
failure. `HPSIM_OUTPUT_DIR` overrides output_dir. Config: JSON, one file:

  {"model": "tiny_cnn" | "alexnet_1col" | {"conv_layers": [...], "fc_layers": [...],
             "input_shape": [C, H, W], "num_classes": L},
   "cluster": {"workers": K, "per_worker_batch": b, "scheme": "A|B|C|DP",
               "variable_batch": false, "seed": 1, "math_mode": "bf16|tf32|f32x3"},
   "hyper": {"momentum": 0.9, "lr": 0.01, "weight_decay": 0.0005, "fc_partial_lr": null},
   "data": {"seed_data": 100, "seed_label": 200}   (per-step seeded N(0,1) batches), or
           {"generator": "gaussian_blobs", "num_examples": N, "seed": s, "separation": sigma}
           (SPEC data_gen, generated on the GPU into the step's device inputs;
           N a multiple of K*b, epochs partition it -- data.py),
   "steps": 5, "output_dir": "out"}

  python -m paper_1404_5997_b200.cli cost-report --config run.json [--json]
      analytical step model (cost_model.py): per-phase table,
      timeline CSV (<output_dir>/timeline.csv: worker,t0,t1,kind,label) and the
      speedup summary vs K=1. Config "cost": {"machine": "b200"|"paper",
      "measured_step_ms": <1-GPU step to calibrate compute to, or null>, plus any
      CostParams field to override}.
"""
from __future__ import annotations

import argparse
import dataclasses
import csv
import json
import os
import sys
import time
from typing import Any, Dict, List

import numpy as np

CSV_HEADER = ["step", "epoch", "loss", "lr", "bytes_fc_activations", "bytes_fc_gradients", "bytes_fc_internal",
              "bytes_conv_sync", "sim_step_time_s", "wall_time_s"]

EXIT_OK, EXIT_VALIDATION, EXIT_RUNTIME, EXIT_EQUIVALENCE = 0, 1, 2, 3
SUSTAINED_BF16_FLOPS = 1.406e15  # MEASURED_PEAKS.json bf16_tflops_sustained (B200)


class ValidationError(Exception):
    pass


# ---------------------------------------------------------------- config
def _specs():
    from . import specs
    return {"tiny_cnn": specs.tiny_cnn, "alexnet_1col": specs.alexnet_1col}


def default_config() -> Dict[str, Any]:
    return {"model": "tiny_cnn",
            "cluster": {"workers": 1, "per_worker_batch": 16, "scheme": "B", "variable_batch": False, "seed": 1,
                        "math_mode": "bf16"},
            "hyper": {"momentum": 0.9, "lr": 0.01, "weight_decay": 0.0005, "fc_partial_lr": None},
            "data": {"seed_data": 100, "seed_label": 200, "generator": None, "num_examples": None, "seed": 0,
                     "separation": 1.0},
            "steps": 5, "output_dir": "out",
            "cost": {"machine": "b200", "measured_step_ms": None}}


def load_config(path: str) -> Dict[str, Any]:
    try:
        with open(path) as fh:
            raw = json.load(fh)
    except (OSError, json.JSONDecodeError) as e:
        raise ValidationError(f"config: cannot read {path}: {e}") from e
    return normalize_config(raw)


def _cost_fields():
    from .cost_model import CostParams
    return {f.name for f in dataclasses.fields(CostParams)}


def normalize_config(raw: Dict[str, Any]) -> Dict[str, Any]:
    """Defaults filled in, field-path validation (SPEC RunConfig invariants)."""
    cfg = default_config()
    if not isinstance(raw, dict):
        raise ValidationError("config: top level must be an object")
    unknown = set(raw) - set(cfg)
    if unknown:
        raise ValidationError(f"config: unknown field(s) {sorted(unknown)}")
    for k, v in raw.items():
        if isinstance(cfg[k], dict) and isinstance(v, dict):
            extra = set(v) - set(cfg[k]) - (_cost_fields() if k == "cost" else set())
            if extra:
                raise ValidationError(f"config.{k}: unknown field(s) {sorted(extra)}")
            cfg[k].update(v)
        else:
            cfg[k] = v
    c = cfg["cluster"]
    if str(c["scheme"]).upper() not in ("A", "B", "C", "DP", "D"):
        raise ValidationError(f"config.cluster.scheme: expected A|B|C|DP, got {c['scheme']!r}")
    if str(c["math_mode"]).lower() not in ("bf16", "tf32", "f32x3"):
        raise ValidationError(f"config.cluster.math_mode: expected bf16|tf32|f32x3, got {c['math_mode']!r}")
    for key in ("workers", "per_worker_batch"):
        if not isinstance(c[key], int) or c[key] < 1:
            raise ValidationError(f"config.cluster.{key}: must be a positive integer")
    if not isinstance(cfg["steps"], int) or cfg["steps"] < 0:
        raise ValidationError("config.steps: must be a non-negative integer")
    if isinstance(cfg["model"], str) and cfg["model"] not in _specs():
        raise ValidationError(f"config.model: unknown preset {cfg['model']!r} (expected {sorted(_specs())})")
    return cfg


def model_spec(cfg):
    from .api import ConvLayerSpec, FcLayerSpec, ModelSpec
    m = cfg["model"]
    if isinstance(m, str):
        return _specs()[m]()
    try:
        return ModelSpec(conv_layers=[ConvLayerSpec(**l) for l in m["conv_layers"]],
                         fc_layers=[FcLayerSpec(**l) for l in m["fc_layers"]],
                         input_shape=list(m["input_shape"]), num_classes=int(m["num_classes"]))
    except (KeyError, TypeError) as e:
        raise ValidationError(f"config.model: {e}") from e


def cluster_config(cfg, **over):
    from .api import ClusterConfig, MathMode, Scheme
    c = dict(cfg["cluster"], **over)
    math = {"bf16": MathMode.BF16, "tf32": MathMode.TF32, "f32x3": MathMode.F32X3}[str(c["math_mode"]).lower()]
    return ClusterConfig(workers=c["workers"], per_worker_batch=c["per_worker_batch"],
                         scheme=Scheme.from_string(str(c["scheme"])), variable_batch=bool(c["variable_batch"]),
                         seed=int(c["seed"]), math_mode=math)


def hyper(cfg):
    from .api import HyperParams
    h = cfg["hyper"]
    return HyperParams(momentum=h["momentum"], lr=h["lr"], weight_decay=h["weight_decay"],
                       fc_partial_lr=h.get("fc_partial_lr"))


def validate(cfg) -> None:
    """Cross-field validation without touching the GPU: the library's geometry
    and config checks (make_geometry, ClusterConfig::validate) via the host-only
    accounting entry; field-path messages as the reference's ConfigError."""
    from .api import ConfigError, HpsimError, step_accounting
    try:
        step_accounting(model_spec(cfg), cluster_config(cfg))
    except ConfigError as e:
        raise ValidationError(str(e)) from e
    except HpsimError as e:
        raise ValidationError(str(e)) from e


def cost_params(cfg):
    from . import cost_model as cm
    c = dict(cfg.get("cost") or {})
    machine = str(c.pop("machine", "b200")).lower()
    c.pop("measured_step_ms", None)
    K = cfg["cluster"]["workers"]
    if machine == "paper":
        params, topo = cm.PAPER, cm.paper_topology(K)
    elif machine == "b200":
        params, topo = cm.b200_params(), cm.b200_topology(K)
    else:
        raise ValidationError(f"config.cost.machine: expected b200|paper, got {machine!r}")
    try:
        params = dataclasses.replace(params, **c)
    except (TypeError, ValueError) as e:
        raise ValidationError(f"config.cost: {e}") from e
    return params, topo


# ---------------------------------------------------------------- checkpoint
def param_tensors(cluster, spec) -> List[tuple]:
    """(name, shape, array) of the gathered model in reference layouts."""
    conv, fc = cluster.gathered_model()
    out = []
    for l, cl in enumerate(spec.conv_layers):
        out.append((f"conv{l}.kernels", [cl.out_channels, cl.in_channels, cl.kernel, cl.kernel], conv[l][0]))
        out.append((f"conv{l}.bias", [cl.out_channels], conv[l][1]))
    for l, fl in enumerate(spec.fc_layers):
        out.append((f"fc{l}.weight", [fl.in_dim, fl.out_dim], fc[l][0]))
        out.append((f"fc{l}.bias", [fl.out_dim], fc[l][1]))
    return out


def write_checkpoint(path: str, tensors: List[tuple]) -> None:
    os.makedirs(path, exist_ok=True)
    manifest = {"format": "raw little-endian float32, one file per tensor (SPEC.md:573)", "precision": "single",
                "tensors": []}
    for name, shape, arr in tensors:
        a = np.ascontiguousarray(np.asarray(arr, dtype="<f4").reshape(shape))
        fn = name + ".f32"
        a.tofile(os.path.join(path, fn))
        manifest["tensors"].append({"name": name, "shape": shape, "dtype": "float32", "file": fn})
    with open(os.path.join(path, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1)


def read_checkpoint(path: str) -> Dict[str, np.ndarray]:
    with open(os.path.join(path, "manifest.json")) as fh:
        man = json.load(fh)
    return {t["name"]: np.fromfile(os.path.join(path, t["file"]), dtype="<f4").reshape(t["shape"])
            for t in man["tensors"]}


# ---------------------------------------------------------------- commands
def dataset_spec(spec, cfg):
    """SPEC data_gen DatasetSpec of the config (None: per-step synthetic batches)."""
    d = cfg["data"]
    if d.get("generator") is None:
        return None
    from .data import DatasetSpec
    if d["generator"] != "gaussian_blobs":
        raise ValidationError(f"config.data.generator: expected gaussian_blobs, got {d['generator']!r}")
    n = d.get("num_examples")
    c = cfg["cluster"]
    kb = c["workers"] * c["per_worker_batch"]
    if not isinstance(n, int) or n < kb or n % kb:
        raise ValidationError(f"config.data.num_examples: expected a positive multiple of K*b = {kb}, got {n!r}")
    if spec.num_classes < 2:
        raise ValidationError("config.data: num_classes must be >= 2 (SPEC.md:502)")
    return DatasetSpec(num_examples=n, input_shape=tuple(spec.input_shape), num_classes=spec.num_classes,
                       seed=int(d.get("seed", 0)), separation=float(d.get("separation", 1.0)))


def batches(spec, cfg, step: int, K: int, b: int):
    from .specs import synthetic_batch
    d = cfg["data"]
    return [synthetic_batch(spec, b, step=step, worker=w, seed_data=d["seed_data"], seed_label=d["seed_label"])
            for w in range(K)]


def cmd_train(cfg, out=None) -> int:
    out = out or sys.stdout
    from .api import Cluster
    spec = model_spec(cfg)
    validate(cfg)
    ds = dataset_spec(spec, cfg)
    outdir = os.environ.get("HPSIM_OUTPUT_DIR", cfg["output_dir"])
    os.makedirs(outdir, exist_ok=True)
    ccfg = cluster_config(cfg)
    K, b = ccfg.workers, ccfg.per_worker_batch
    hp = hyper(cfg)
    from .specs import algorithmic_gemm_flops
    sim_s = algorithmic_gemm_flops(spec, b, K) / SUSTAINED_BF16_FLOPS
    with open(os.path.join(outdir, "metrics.csv"), "w", newline="") as fh:
        wr = csv.writer(fh)
        wr.writerow(CSV_HEADER)
        if cfg["steps"] > 0:
            cluster = Cluster(spec, ccfg)
            feed = None
            if ds is not None:  # the input pipeline: batches generated on the GPU
                from .data import DeviceBatches
                feed = DeviceBatches(ds, K, b)
            for s in range(cfg["steps"]):
                t0 = time.perf_counter()
                if feed is not None:
                    xs, ts = feed.batches(s, stream=cluster.stream_ptr())
                    r = cluster.run_step(xs, ts, hp, device=True)
                else:
                    xb = batches(spec, cfg, s, K, b)
                    t0 = time.perf_counter()
                    r = cluster.run_step([x for x, _ in xb], [t for _, t in xb], hp)
                wall = time.perf_counter() - t0
                m = r.metrics
                # sim_step_time_s: deterministic model time of the step on one
                # B200 -- algorithmic GEMM FLOPs at the measured sustained bf16
                # rate (the B200 path has no cost-model simulation; the measured
                # device time is nondeterministic and goes to the log instead)
                epoch = (s * K * b) // ds.num_examples if ds is not None else 0
                wr.writerow([s, epoch, repr(float(m.loss)), repr(float(hp.lr))] + [int(v) for v in m.bytes_sent] +
                            [repr(sim_s), f"{wall:.6f}"])
            write_checkpoint(os.path.join(outdir, "checkpoint"), param_tensors(cluster, spec))
            cluster.close()
    print(f"train: {cfg['steps']} steps -> {outdir}/metrics.csv", file=out)
    return EXIT_OK


def cmd_verify_equivalence(cfg, tol: float = 2e-5, skip_broadcast: bool = False, out=None) -> int:
    """Schemes A/B/C (exact) vs one worker on the concatenated K*b batch, all on
    B200 with 3xTF32 parity math; max relative divergence per parameter tensor."""
    out = out or sys.stdout
    from .api import Cluster
    spec = model_spec(cfg)
    validate(cfg)
    c = cfg["cluster"]
    K, b = c["workers"], c["per_worker_batch"]
    steps = max(1, cfg["steps"])
    hp = hyper(cfg)
    if c.get("variable_batch"):
        raise ValidationError("verify-equivalence: variable_batch must be false (SPEC.md:548)")

    def run(workers, batch, scheme, data):
        cl = Cluster(spec, cluster_config(cfg, workers=workers, per_worker_batch=batch, scheme=scheme,
                                          variable_batch=False, math_mode="f32x3"))
        if skip_broadcast and workers > 1:
            cl.set_skip_sync_broadcast(True)
        for s in range(steps):
            xs, ts = data(s)
            cl.run_step(xs, ts, hp)
        # per-worker parameters: conv replicas and the pasted FC shards of every worker
        res = [param_tensors(cl, spec)]
        for w in range(1, workers):
            res.append([(f"{n}@worker{w}", sh, cl.param(w, which, l)) for n, sh, which, l in
                        [(f"conv{l}.kernels", None, 0, l) for l in range(len(spec.conv_layers))] +
                        [(f"conv{l}.bias", None, 1, l) for l in range(len(spec.conv_layers))]])
        cl.close()
        return res

    def split_data(s):
        xb = batches(spec, cfg, s, K, b)
        return [x for x, _ in xb], [t for _, t in xb]

    def joint_data(s):
        xb = batches(spec, cfg, s, K, b)
        return [np.concatenate([x for x, _ in xb])], [np.concatenate([t for _, t in xb])]

    oracle = run(1, K * b, "A", joint_data)[0]
    ref = {n: np.asarray(a, dtype=np.float64).ravel() for n, _, a in oracle}
    worst_all = 0.0
    failed = []
    for scheme in ("A", "B", "C"):
        if scheme == "C" and b % K:
            print(f"scheme C: skipped (b={b} not divisible by K={K})", file=out)
            continue
        got = run(K, b, scheme, split_data)
        worst, where = 0.0, None
        for n, _, a in got[0]:
            r = ref[n]
            d = float(np.abs(np.asarray(a, dtype=np.float64).ravel() - r).max() / max(np.abs(r).max(), 1e-30))
            if d > worst:
                worst, where = d, n
        for extra in got[1:]:  # every worker's conv replica must match too
            for n, _, a in extra:
                base = n.split("@")[0]
                r = ref[base]
                d = float(np.abs(np.asarray(a, dtype=np.float64).ravel() - r).max() / max(np.abs(r).max(), 1e-30))
                if d > worst:
                    worst, where = d, n
        worst_all = max(worst_all, worst)
        status = "ok" if worst <= tol else "FAIL"
        print(f"scheme {scheme}: max relative divergence {worst:.3e} ({where}) {status}", file=out)
        if worst > tol:
            failed.append((scheme, where, worst))
    if failed:
        print("verify-equivalence: divergence above tolerance " + ", ".join(
            f"{s}:{w} {d:.3e}" for s, w, d in failed), file=out)
        return EXIT_EQUIVALENCE
    print(f"verify-equivalence: all schemes within {tol:g} (max {worst_all:.3e})", file=out)
    return EXIT_OK


def cmd_cost_report(cfg, as_json: bool = False, out=None) -> int:
    """per-phase table + timeline CSV + speedup summary."""
    from . import cost_model as cm
    out = out or sys.stdout
    validate(cfg)
    spec, cl = model_spec(cfg), cluster_config(cfg)
    params, topo = cost_params(cfg)
    meas = (cfg.get("cost") or {}).get("measured_step_ms")
    scale = cm.calibrate(spec, cl.per_worker_batch, params, meas * 1e-3) if meas else 1.0
    r = cm.speedup(spec, cl, topo, params, compute_scale=scale)
    tl = r.pop("timeline")
    odir = os.environ.get("HPSIM_OUTPUT_DIR", cfg["output_dir"])
    os.makedirs(odir, exist_ok=True)
    with open(os.path.join(odir, "timeline.csv"), "w") as fh:
        fh.write(tl.csv())
    summary = {"workers": cl.workers, "per_worker_batch": cl.per_worker_batch, "scheme": cl.scheme.name,
               "compute_scale": scale, "phases_s": tl.phase_table(), "internal_s": tl.internal_s,
               "sync_s": tl.sync_s, "sync_exposed_s": tl.sync_exposed_s, **r}
    if as_json:
        print(json.dumps(summary, sort_keys=True), file=out)
        return EXIT_OK
    print(f"cost-report: K={cl.workers} b={cl.per_worker_batch} scheme={cl.scheme.name} "
          f"flops/s={params.flops_per_sec:.4g}x{scale:.3f} link={params.link_bandwidth:.4g} B/s", file=out)
    print(f"{'phase':<12}{'seconds':>14}", file=out)
    for k, v in tl.phase_table().items():
        print(f"{k:<12}{v:>14.6e}", file=out)
    h = r["hidden_comm_fraction"]
    print(f"step_time_s={r['step_time_K']:.6e} speedup={r['speedup']:.4f} images/s={r['images_per_s']:.1f} "
          f"hidden_comm_fraction={'n/a' if h is None else f'{h:.6f}'}", file=out)
    return EXIT_OK


def main(argv=None) -> int:
    p = argparse.ArgumentParser(prog="python -m paper_1404_5997_b200.cli")
    sub = p.add_subparsers(dest="cmd", required=True)
    for name in ("train", "verify-equivalence", "cost-report"):
        s = sub.add_parser(name)
        s.add_argument("--config", required=True)
        s.add_argument("--seed", type=int, default=None)
        s.add_argument("--json", action="store_true")
        if name == "verify-equivalence":
            s.add_argument("--tol", type=float, default=2e-5)
            s.add_argument("--skip-broadcast", action="store_true")
    a = p.parse_args(argv)
    try:
        cfg = load_config(a.config)
        if a.seed is not None:
            cfg["cluster"]["seed"] = a.seed
        if a.cmd == "train":
            return cmd_train(cfg)
        if a.cmd == "cost-report":
            return cmd_cost_report(cfg, a.json)
        return cmd_verify_equivalence(cfg, tol=a.tol, skip_broadcast=a.skip_broadcast)
    except ValidationError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_VALIDATION
    except Exception as e:  # runtime (CUDA / NCCL / IO)
        from .api import ConfigError
        if isinstance(e, ConfigError):
            print(f"error: {e}", file=sys.stderr)
            return EXIT_VALIDATION
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_RUNTIME


if __name__ == "__main__":
    sys.exit(main())
