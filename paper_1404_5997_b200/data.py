"""Input pipeline: SPEC `data_gen` on the GPU.

The reference specifies the dataset generator (class-conditional Gaussian
blobs, one-hot targets, bit-reproducible per (spec, seed), class counts within
+-1 of N/L, L < 2 is a configuration error) but ships no code for it; the
generator itself is defined in csrc/datagen.cu and include/hpsim_b200.h
(hp_data_generate). Batches are generated straight into device memory and fed
to Cluster.run_step(..., device=True): the input never crosses PCIe.

Epoch batching ("partitions examples without overlap or omission
per epoch"): step s, worker w of a K-worker, b-per-worker run takes examples
[((s * K + w) * b) mod N, + b); N must be a multiple of K*b.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from ._lib import HpDatasetSpec, lib
from .api import ConfigError, _check


@dataclass
class DatasetSpec:
    """SPEC.md:492 DatasetSpec: num_examples, input_shape C x H x W, num_classes L,
    seed, generator gaussian_blobs; separation = std of the class means."""
    num_examples: int
    input_shape: Tuple[int, int, int]
    num_classes: int
    seed: int = 0
    separation: float = 1.0
    generator: str = "gaussian_blobs"

    def _c(self) -> HpDatasetSpec:
        if self.generator != "gaussian_blobs":
            raise ConfigError(f"data.generator: unknown generator '{self.generator}' (gaussian_blobs)")
        c, h, w = self.input_shape
        return HpDatasetSpec(int(self.num_examples), int(c), int(h), int(w), int(self.num_classes),
                             int(self.seed) & 0xFFFFFFFFFFFFFFFF, float(self.separation))

    @property
    def example_size(self) -> int:
        c, h, w = self.input_shape
        return int(c) * int(h) * int(w)


def generate(spec: DatasetSpec, first: int = 0, count: int = -1, device: bool = True, stream=None):
    """Examples [first, first + count) (count -1: to the end) as (inputs [count][C][H][W],
    targets [count][L]) float32: torch CUDA tensors (device=True, generated on the
    current device, ordered on `stream` / the current stream) or numpy arrays."""
    cs = spec._c()
    if count < 0:
        count = spec.num_examples - first
    c, h, w = spec.input_shape
    if device:
        import torch
        x = torch.empty((max(count, 0), c, h, w), dtype=torch.float32, device="cuda")
        t = torch.empty((max(count, 0), spec.num_classes), dtype=torch.float32, device="cuda")
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        _check(lib.hp_data_generate(C.byref(cs), first, count, x.data_ptr() if count > 0 else None,
                                    t.data_ptr() if count > 0 else None, 1, C.c_void_p(st)))
        return x, t
    x = np.empty((max(count, 0), c, h, w), dtype=np.float32)
    t = np.empty((max(count, 0), spec.num_classes), dtype=np.float32)
    _check(lib.hp_data_generate(C.byref(cs), first, count, x.ctypes.data if count > 0 else None,
                                t.ctypes.data if count > 0 else None, 0, None))
    return x, t


def class_of(spec: DatasetSpec, index: int) -> int:
    """The class of example `index` (host evaluation of the same permutation)."""
    r = C.c_int64(-1)
    _check(lib.hp_data_class_of(C.byref(spec._c()), int(index), C.byref(r)))
    return int(r.value)


def epoch_ranges(num_examples: int, workers: int, per_worker_batch: int, step: int) -> List[Tuple[int, int]]:
    """[first, first + b) of each worker at `step` (module docstring)."""
    kb = workers * per_worker_batch
    if num_examples < kb or num_examples % kb:
        raise ConfigError(f"data.num_examples: {num_examples} must be a positive multiple of K*b = {kb} "
                          "(epochs partition the examples into whole steps)")
    base = (step * kb) % num_examples
    return [(base + w * per_worker_batch, per_worker_batch) for w in range(workers)]


class DeviceBatches:
    """Per-step device batches for a Cluster: batches(step) -> ([x_w], [t_w]) torch
    tensors, generated into two alternating buffer sets (the next step's batch can be
    generated while the current one trains)."""

    def __init__(self, spec: DatasetSpec, workers: int, per_worker_batch: int):
        import torch
        self.spec, self.K, self.b = spec, workers, per_worker_batch
        epoch_ranges(spec.num_examples, workers, per_worker_batch, 0)  # validates N
        c, h, w = spec.input_shape
        self._x = [[torch.empty((per_worker_batch, c, h, w), device="cuda") for _ in range(workers)] for _ in range(2)]
        self._t = [[torch.empty((per_worker_batch, spec.num_classes), device="cuda") for _ in range(workers)]
                   for _ in range(2)]

    def batches(self, step: int, stream=None):
        import torch
        slot = step & 1
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        cs = self.spec._c()
        for w, (first, n) in enumerate(epoch_ranges(self.spec.num_examples, self.K, self.b, step)):
            _check(lib.hp_data_generate(C.byref(cs), first, n, self._x[slot][w].data_ptr(),
                                        self._t[slot][w].data_ptr(), 1, C.c_void_p(st)))
        return list(self._x[slot]), list(self._t[slot])
