"""Golden first-step fixtures for the BENCHMARKED configuration (test infrastructure).

The double-precision oracle (oracle/hpsim_oracle.c, itself pinned bit-exactly
to the compiled reference in tests/test_oracle_vs_reference.py and torch-checked
for the LRN / pool superset in tests/test_oracle_extensions.py) runs one
AlexNet-1col training step at the bench's own shapes:

  k1b  K=1, scheme B, exact SGD, b=128          (configs[2] at N=1 -- bench.py's step)
  k2c  K=2, scheme C, approximate (variable), b=128 per worker  (configs[3]'s mode)

each with the oracle in plain double (the reference restatement) and in
bf16-storage mode (k1bq / k2cq: tensors rounded to bf16 exactly where the
B200 bf16 math mode stores them, so pool argmax and ReLU decisions are taken on
the same values -- see oracle/hpsim_oracle.c), on the same seeded synthetic inputs the product generates (specs.synthetic_batch,
GaussianSampler replay) and the same initial weights (init_model replay). A full
AlexNet step costs the oracle minutes of CPU, so the result is committed: per
parameter tensor, the max |value| over the FULL tensor and the values at a fixed
pseudo-random sample of indices (all of them for tensors up to SAMPLE entries),
for the momenta after step 1 (pure gradient history: -lr*(g + wd*w0) in exact
mode) and the loss. tests/test_alexnet_parity_gpu.py replays the step on the
B200 and compares.

Run (here, ~15 min on 8 cores):  python tests/golden/make_alexnet_golden.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_1404_5997_b200 as hp  # noqa: E402

SAMPLE = 131072
PRIME = 2654435761  # > every tensor size here, so the strided sample has no repeats
HYPER = (0.9, 0.01, 5e-4)  # momentum, lr, weight decay
CASES = {"k1b": (1, "B", False, "double"), "k2c": (2, "C", True, "double"),
         "k1bq": (1, "B", False, "bf16"), "k2cq": (2, "C", True, "bf16")}
B = 128
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "alexnet_step1.npz")


def sample_index(n: int) -> np.ndarray:
    if n <= SAMPLE:
        return np.arange(n, dtype=np.int64)
    return (np.arange(SAMPLE, dtype=np.int64) * PRIME) % n


def main(only=None):
    spec = hp.alexnet_1col()
    out = dict(np.load(OUT)) if os.path.exists(OUT) else {}
    out["hyper"] = np.array(HYPER)
    out["b"] = np.array([B])
    for name, (K, scheme, var, storage) in CASES.items():
        if only and name not in only:
            continue
        t0 = time.time()
        o = O.OracleCluster(spec, workers=K, per_worker_batch=B, scheme=scheme, variable_batch=var,
                            precision="single", seed=1)
        o.set_storage_rounding(storage)
        xs, ts = zip(*[hp.synthetic_batch(spec, B, step=0, worker=w) for w in range(K)])
        m = o.run_step([x.astype(np.float64) for x in xs], [t.astype(np.float64) for t in ts],
                       O.make_hyper_c(*HYPER))
        out[f"{name}_loss"] = np.array([m.loss])
        nconv, nfc = len(spec.conv_layers), len(spec.fc_layers)
        for w in range(K):
            for which in (4, 5, 6, 7):
                for l in range(nconv if which in (4, 5) else nfc):
                    if which in (4, 5) and w > 0:
                        continue  # conv replicas are identical after the sync
                    v = o.param(w, which, l)
                    key = f"{name}_w{w}_p{which}_l{l}"
                    out[key + "_max"] = np.array([np.abs(v).max()])
                    out[key + "_val"] = v[sample_index(v.size)].astype(np.float32)
                    out[key + "_n"] = np.array([v.size])
        print(f"{name}: loss {m.loss:.10f} ({time.time() - t0:.0f} s)", flush=True)
        np.savez_compressed(OUT, **out)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
