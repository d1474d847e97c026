"""Network specs and seeded synthetic data for the configs in BASELINE.json.

* tiny_cnn(): the CPU oracle's default workload: 3x32x32 ->
  conv 3->32 k5 p2 -> conv 32->32 k4 s2 p1 -> conv 32->64 k4 s2 p1 -> 4096 ->
  fc 256 ReLU -> fc 10. Expressible by the reference as is.
* alexnet_1col(): Krizhevsky's one-column AlexNet: filters
  64/192/384/384/256, conv1 11x11/4 p2 (floor) -> LRN -> pool 3/2, conv2 5x5
  p2 -> LRN -> pool, conv3-5 3x3 p1, pool -> 9216 -> 4096 -> 4096 -> 1000
  independent logistic units. Needs the floor/LRN/pool superset.
* alexnet_standin_227(): the stride-only stand-in the reference itself accepts
  (SURVEY.md A.5): identical parameter counts and 9216-wide boundary.

Synthetic data: pixels N(0,1) NCHW from
GaussianSampler(seed_data + 7919*step + worker); labels uniform over L from
mt19937_64(seed_label + 7919*step + worker) (top 64 bits mod L), one-hot.
"""
from __future__ import annotations

import numpy as np

from .api import ConvLayerSpec, FcLayerSpec, ModelSpec, gaussian_f32

LRN = dict(lrn_size=5, lrn_alpha=1e-4, lrn_beta=0.75, lrn_k=2.0)


def tiny_cnn() -> ModelSpec:
    return ModelSpec(
        conv_layers=[ConvLayerSpec(3, 32, 5, 1, 2), ConvLayerSpec(32, 32, 4, 2, 1), ConvLayerSpec(32, 64, 4, 2, 1)],
        fc_layers=[FcLayerSpec(4096, 256, True), FcLayerSpec(256, 10, False)],
        input_shape=[3, 32, 32], num_classes=10)


def alexnet_1col(num_classes: int = 1000) -> ModelSpec:
    return ModelSpec(
        conv_layers=[
            ConvLayerSpec(3, 64, 11, 4, 2, floor_mode=True, pool_kernel=3, pool_stride=2, **LRN),
            ConvLayerSpec(64, 192, 5, 1, 2, pool_kernel=3, pool_stride=2, **LRN),
            ConvLayerSpec(192, 384, 3, 1, 1),
            ConvLayerSpec(384, 384, 3, 1, 1),
            ConvLayerSpec(384, 256, 3, 1, 1, pool_kernel=3, pool_stride=2),
        ],
        fc_layers=[FcLayerSpec(9216, 4096, True), FcLayerSpec(4096, 4096, True),
                   FcLayerSpec(4096, num_classes, False)],
        input_shape=[3, 224, 224], num_classes=num_classes)


def alexnet_standin_227() -> ModelSpec:
    return ModelSpec(
        conv_layers=[ConvLayerSpec(3, 64, 11, 4, 0), ConvLayerSpec(64, 192, 5, 2, 1),
                     ConvLayerSpec(192, 384, 3, 2, 0), ConvLayerSpec(384, 384, 3, 1, 1),
                     ConvLayerSpec(384, 256, 3, 2, 0)],
        fc_layers=[FcLayerSpec(9216, 4096, True), FcLayerSpec(4096, 4096, True), FcLayerSpec(4096, 1000, False)],
        input_shape=[3, 227, 227], num_classes=1000)


def mt19937_64(seed: int, n: int) -> np.ndarray:
    """std::mt19937_64(seed), n outputs (pure numpy; integer-exact)."""
    N, M = 312, 156
    mask = (1 << 64) - 1
    mt = [0] * N
    mt[0] = seed & mask
    for i in range(1, N):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & mask
    out = np.empty(n, dtype=np.uint64)
    idx = N
    for k in range(n):
        if idx >= N:
            for i in range(N):
                x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % N] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[i] = mt[(i + M) % N] ^ xa
            idx = 0
        x = mt[idx]
        idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000 & mask
        x ^= (x << 37) & 0xFFF7EEE000000000 & mask
        x ^= x >> 43
        out[k] = x
    return out


def synthetic_batch(spec: ModelSpec, b: int, step: int = 0, worker: int = 0, seed_data: int = 100,
                    seed_label: int = 200):
    """(images [b][C][H][W] float32, one-hot targets [b][L] float32)."""
    c, h, w = spec.input_shape
    x = gaussian_f32(seed_data + 7919 * step + worker, b * c * h * w).reshape(b, c, h, w)
    labels = (mt19937_64(seed_label + 7919 * step + worker, b) % np.uint64(spec.num_classes)).astype(np.int64)
    t = np.zeros((b, spec.num_classes), dtype=np.float32)
    t[np.arange(b), labels] = 1.0
    return x, t


def algorithmic_gemm_flops(spec: ModelSpec, b: int, workers: int = 1) -> float:
    """Algorithmic GEMM FLOPs of one step on one worker:
    conv fprop + wgrad + dgrad (conv1 dgrad excluded: the reference discards it),
    2 FLOPs per MAC on the useful problem (no padded channels, taps or border
    rows); the FC stack's 3 GEMMs over K*b examples split K ways."""
    c, h, w = spec.input_shape
    total = 0.0
    for i, l in enumerate(spec.conv_layers):
        def od(x):
            return (x + 2 * l.pad - l.kernel) // l.stride + 1
        oh, ow = od(h), od(w)
        macs = b * oh * ow * l.out_channels * l.kernel * l.kernel * l.in_channels
        total += 2.0 * macs * (2 if i == 0 else 3)
        c, h, w = l.out_channels, oh, ow
        if l.pool_kernel:
            h = (h - l.pool_kernel) // l.pool_stride + 1
            w = (w - l.pool_kernel) // l.pool_stride + 1
    for f in spec.fc_layers:
        total += 3 * 2.0 * b * f.in_dim * f.out_dim
    return total
