"""Kernel variants that must agree bit for bit (GPU). The flat shuffle-halo
LRN+pool kernels (conv1: 8-channel vectors, conv2: 12-channel vectors) are the
default; HP_DEV_LRN_BWD_SMEM=1 / HP_DEV_LRN_FWD_SMEM=1 select the smem kernels
they replaced. The switch is read once per process, so each variant runs an
AlexNet-1col bf16 step sequence in its own subprocess and the parameter bytes
are compared."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_1404_5997_b200 as hp
spec = hp.alexnet_1col()
c = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=32, seed=5, math_mode=hp.MathMode.{math}))
for s in range(2):
    x, t = hp.synthetic_batch(spec, 32, step=s)
    r = c.run_step([x], [t], hp.HyperParams(momentum=0.9, lr=1e-3, weight_decay=5e-4))
h = hashlib.sha256()
for which in range(4):
    for l in range(len(spec.conv_layers) if which < 2 else len(spec.fc_layers)):
        h.update(np.ascontiguousarray(c.param(0, which, l)).tobytes())
print(repr(r.metrics.loss), h.hexdigest())
"""


def run(env_extra, math):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, math=math)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return out.stdout.strip().splitlines()[-1]


@pytest.mark.gpu
@pytest.mark.parametrize("math", ["BF16", "F32X3"])
def test_flat_lrn_kernels_match_smem_kernels(math):
    flat = run({}, math)
    assert flat == run({"HP_DEV_LRN_BWD_SMEM": "1"}, math)
    assert flat == run({"HP_DEV_LRN_FWD_SMEM": "1"}, math)
