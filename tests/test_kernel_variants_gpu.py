"""Kernel variants that must agree bit for bit (GPU). The window-tile LRN+pool
forward (LRN once per conv pixel into an smem tile, pooled from smem) and the
quad backward (2x2 conv pixels per thread sharing their 4 candidate windows)
are the default; HP_DEV_LRN_FWD_SMEM=1 / HP_DEV_LRN_BWD_SMEM=1 select the
smem-band kernels, which use the same pinned LRN arithmetic (kernels.cu
lrn_scale5 / lrn_bwd_out) and window order. The switch is read once per
process, so each variant runs one AlexNet-1col step in its own subprocess and
every parameter tensor is compared bit for bit."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_1404_5997_b200 as hp
spec = hp.alexnet_1col()
c = hp.Cluster(spec, hp.ClusterConfig(workers=1, per_worker_batch=32, seed=5, math_mode=hp.MathMode.{math}))
x, t = hp.synthetic_batch(spec, 32, step=0)
r = c.run_step([x], [t], hp.HyperParams(momentum=0.9, lr=1e-3, weight_decay=5e-4))
out = {{"loss": r.metrics.loss, "hash": {{}}, "conv_b": {{}}}}
for which in range(4):
    for l in range(len(spec.conv_layers) if which < 2 else len(spec.fc_layers)):
        v = np.ascontiguousarray(c.param(0, which, l))
        out["hash"][f"{{which}}_{{l}}"] = hashlib.sha256(v.tobytes()).hexdigest()
        if which == 1:
            out["conv_b"][str(l)] = v.astype(float).tolist()
print(json.dumps(out))
"""


def run(env_extra, math):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, math=math)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("math", ["BF16", "F32X3"])
def test_tile_quad_lrn_kernels_match_smem_kernels(math):
    rows = run({}, math)
    for env in ({"HP_DEV_LRN_FWD_SMEM": "1"}, {"HP_DEV_LRN_BWD_SMEM": "1"}):
        alt = run(env, math)
        assert alt["loss"] == rows["loss"], env
        for k, h in rows["hash"].items():
            assert alt["hash"][k] == h, (env, k)
