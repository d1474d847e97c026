"""Python mirror of the reference's hpsim interface, over the C ABI.

Names, fields and error behaviour follow /root/reference/proj/core/include/hpsim
(ModelSpec / ConvLayerSpec / FcLayerSpec: model.hpp:24-58; ClusterConfig /
Cluster / StepMetrics / StepTrace: cluster.hpp:36-212; HyperParams:
optimizer.hpp:27-51; the four exception types: errors.hpp:22-44). The step
itself runs entirely in libhpsim_b200.so (CUDA, sm_100a); this module only
marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from ._lib import (HpClusterConfig, HpConvLayer, HpFcLayer, HpGemmProf, HpHyper, HpModelSpec,
                   HpStepMetrics, HpTraceEvent, last_error, lib)


# ---------------------------------------------------------------- errors
class HpsimError(RuntimeError):
    code = 0


class ConfigError(HpsimError):
    """A spec, cluster, or run configuration is invalid (errors.hpp:29-32)."""
    code = 1


class DimensionError(HpsimError):
    """Tensor shapes or precisions do not line up (errors.hpp:22-26)."""
    code = 2


class DomainError(HpsimError):
    """A numeric argument is outside the operation's domain (errors.hpp:35-38)."""
    code = 3


class UsageError(HpsimError):
    """An API was called out of contract (errors.hpp:41-44)."""
    code = 4


class CudaError(HpsimError):
    code = 5


class NcclError(HpsimError):
    code = 6


_ERRORS = {1: ConfigError, 2: DimensionError, 3: DomainError, 4: UsageError, 5: CudaError, 6: NcclError}


def _check(rc: int) -> None:
    if rc != 0:
        raise _ERRORS.get(rc, HpsimError)(last_error())


# ---------------------------------------------------------------- enums
class Scheme(enum.IntEnum):
    A = 0
    B = 1
    C = 2
    DP = 3  # B200 extension: pure data parallelism (FC replicated, gradients all-reduced)

    @staticmethod
    def from_string(s: str) -> "Scheme":  # cluster.cpp:31-36
        if s in ("A", "a"):
            return Scheme.A
        if s in ("B", "b"):
            return Scheme.B
        if s in ("C", "c"):
            return Scheme.C
        if s in ("DP", "dp", "D", "d"):
            return Scheme.DP
        raise ConfigError(f"unknown scheme '{s}' (expected A|B|C)")


class Precision(enum.IntEnum):
    SINGLE = 0
    DOUBLE = 1


class MathMode(enum.IntEnum):
    BF16 = 0
    TF32 = 1
    F32X3 = 2


class Transport(enum.IntEnum):
    LOGICAL = 0
    NCCL = 1


class Phase(enum.IntEnum):
    CONV_FWD = 0
    FC_FWD = 1
    FC_BWD = 2
    CONV_BWD = 3
    SYNC = 4


class MsgClass(enum.IntEnum):
    FC_ACTIVATIONS = 0
    FC_GRADIENTS = 1
    FC_INTERNAL = 2
    CONV_SYNC = 3


# ---------------------------------------------------------------- specs
@dataclass
class ConvLayerSpec:
    in_channels: int
    out_channels: int
    kernel: int
    stride: int = 1
    pad: int = 0
    relu: bool = True
    # superset (AlexNet); absent from the reference
    floor_mode: bool = False
    lrn_size: int = 0
    lrn_alpha: float = 0.0
    lrn_beta: float = 0.0
    lrn_k: float = 0.0
    pool_kernel: int = 0
    pool_stride: int = 0


@dataclass
class FcLayerSpec:
    in_dim: int
    out_dim: int
    relu: bool = False


@dataclass
class ModelSpec:
    conv_layers: List[ConvLayerSpec]
    fc_layers: List[FcLayerSpec]
    input_shape: List[int]
    num_classes: int

    def conv_output_sizes(self):
        out = []
        h, w = self.input_shape[1], self.input_shape[2]
        for l in self.conv_layers:
            def od(x):
                num = x + 2 * l.pad - l.kernel
                if num < 0 or (not l.floor_mode and num % l.stride):
                    raise ConfigError("conv: output dimension is not a positive integer")
                return num // l.stride + 1
            h, w = od(h), od(w)
            if l.pool_kernel:
                h, w = (h - l.pool_kernel) // l.pool_stride + 1, (w - l.pool_kernel) // l.pool_stride + 1
            out.append((h, w))
        return out

    def flattened_conv_size(self) -> int:
        h, w = self.conv_output_sizes()[-1]
        return self.conv_layers[-1].out_channels * h * w


@dataclass
class ClusterConfig:
    workers: int = 1
    per_worker_batch: int = 128
    scheme: Scheme = Scheme.B
    variable_batch: bool = False
    precision: Precision = Precision.SINGLE
    seed: int = 0
    # B200 fields
    math_mode: MathMode = MathMode.BF16
    transport: Transport = Transport.LOGICAL
    rank: int = 0
    device: int = -1
    nccl_id: Optional[bytes] = None


@dataclass
class HyperParams:
    momentum: float = 0.9
    lr: float = 0.01
    weight_decay: float = 0.0
    fc_partial_lr: Optional[float] = None


@dataclass
class TraceEvent:
    phase: Phase
    sub_batch: int
    worker: int
    bytes_total: int
    bytes_max_sender: int


@dataclass
class StepMetrics:
    loss: float
    fc_update_count: int
    conv_update_count: int
    bytes_sent: List[int]


@dataclass
class StepResult:
    metrics: StepMetrics
    trace: List[TraceEvent] = field(default_factory=list)


def _spec_c(spec: ModelSpec):
    convs = (HpConvLayer * len(spec.conv_layers))()
    for i, l in enumerate(spec.conv_layers):
        convs[i] = HpConvLayer(l.in_channels, l.out_channels, l.kernel, l.stride, l.pad, int(bool(l.relu)),
                               int(bool(l.floor_mode)), l.lrn_size, l.lrn_alpha, l.lrn_beta, l.lrn_k,
                               l.pool_kernel, l.pool_stride)
    fcs = (HpFcLayer * len(spec.fc_layers))()
    for i, l in enumerate(spec.fc_layers):
        fcs[i] = HpFcLayer(l.in_dim, l.out_dim, int(bool(l.relu)))
    s = HpModelSpec()
    s.conv = C.cast(convs, C.POINTER(HpConvLayer))
    s.n_conv = len(spec.conv_layers)
    s.fc = C.cast(fcs, C.POINTER(HpFcLayer))
    s.n_fc = len(spec.fc_layers)
    for i in range(3):
        s.input_shape[i] = spec.input_shape[i]
    s.num_classes = spec.num_classes
    return s, (convs, fcs)


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(lib.hp_nccl_unique_id(C.byref(buf)))
    return bytes(buf)


def _ptr(x) -> int:
    """Address of a host numpy array or a torch tensor (float32, contiguous)."""
    if isinstance(x, np.ndarray):
        if x.dtype != np.float32 or not x.flags["C_CONTIGUOUS"]:
            raise DimensionError("host tensors must be C-contiguous float32")
        return x.ctypes.data
    if str(getattr(x, "dtype", "")) != "torch.float32" or not x.is_contiguous():
        raise DimensionError("tensors must be contiguous float32")
    return int(x.data_ptr())


def _on_device(x) -> bool:
    """HP_MEM_DEVICE for CUDA tensors; numpy arrays and (pinned) CPU tensors are host memory."""
    return bool(getattr(x, "is_cuda", False))


def _shape_str(shape) -> str:  # shape_string (tensor.cpp:57-66)
    return "[" + "x".join(str(int(d)) for d in shape) + "]"


class Cluster:
    """hpsim::Cluster on B200 (cluster.hpp:178-212)."""

    def __init__(self, spec: ModelSpec, config: ClusterConfig):
        self.spec = spec
        self.config = config
        sc, self._keep = _spec_c(spec)
        cfg = HpClusterConfig()
        cfg.workers = config.workers
        cfg.per_worker_batch = config.per_worker_batch
        cfg.scheme = int(config.scheme)
        cfg.variable_batch = int(bool(config.variable_batch))
        cfg.precision = int(config.precision)
        cfg.seed = config.seed
        cfg.math_mode = int(config.math_mode)
        cfg.transport = int(config.transport)
        cfg.rank = config.rank
        cfg.device = config.device
        if config.nccl_id is not None:
            C.memmove(cfg.nccl_id, config.nccl_id, 128)
        h = C.c_void_p()
        _check(lib.hp_cluster_create(C.byref(sc), C.byref(cfg), C.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.hp_cluster_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def workers(self) -> int:
        return self.config.workers

    def run_step(self, batches: Sequence, targets: Sequence, hp: HyperParams, lr: Optional[float] = None,
                 device: Optional[bool] = None) -> StepResult:
        """One training step (cluster.cpp:439-711). batches[i]: [b][C][H][W] float32,
        targets[i]: [b][L]; host numpy arrays or device tensors (all the same kind)."""
        lr = hp.lr if lr is None else lr
        n = len(batches)
        k = 1 if self.config.transport == Transport.NCCL else self.config.workers
        if n != k or len(targets) != k:  # cluster.cpp:444-450
            raise UsageError(f"run_step: expected {k} batches and targets, got {n} / {len(targets)}")
        self._check_inputs(batches, targets, "run_step")
        kinds = {_on_device(x) for x in list(batches) + list(targets)}
        if len(kinds) != 1:
            raise UsageError("run_step: batches and targets must all be host or all be device memory")
        if device is None:
            device = kinds.pop()
        elif bool(device) != kinds.pop():
            raise UsageError("run_step: device= does not match where the tensors live")
        bp = (C.c_void_p * n)(*[_ptr(x) for x in batches])
        tp = (C.c_void_p * n)(*[_ptr(t) for t in targets])
        h = HpHyper(hp.momentum, hp.lr, hp.weight_decay, 0 if hp.fc_partial_lr is None else 1,
                    0.0 if hp.fc_partial_lr is None else hp.fc_partial_lr)
        m = HpStepMetrics()
        _check(lib.hp_cluster_run_step(self._h, bp, tp, 1 if device else 0, C.byref(h), lr, C.byref(m)))
        return StepResult(StepMetrics(m.loss, m.fc_update_count, m.conv_update_count, list(m.bytes_sent)),
                          self.trace())

    def _check_inputs(self, batches: Sequence, targets: Sequence, fn: str) -> None:
        """Full shapes before any native call: rows (UsageError, cluster.cpp:451-457),
        then [b][C][H][W] (DimensionError, model.cpp:204-214) and [b][L]
        (logistic_xent's shape check, tensor.cpp:172-182). The native side reads
        exactly b*C*H*W and b*L floats per worker."""
        b = self.config.per_worker_batch
        C_, H, W = self.spec.input_shape
        L = self.spec.num_classes
        for i, (x, t) in enumerate(zip(batches, targets)):
            if x.shape[0] != b or t.shape[0] != b:
                raise UsageError(f"{fn}: worker {i} batch must hold exactly {b} examples")
            if len(x.shape) != 4 or tuple(x.shape[1:]) != (C_, H, W):
                raise DimensionError(f"forward: batch shape {_shape_str(x.shape)} does not match model input "
                                     f"[Bx{C_}x{H}x{W}]")
            if tuple(t.shape) != (b, L):
                raise DimensionError(f"logistic_xent: shape mismatch {_shape_str((b, L))} vs {_shape_str(t.shape)}")

    def prefetch(self, batches: Sequence, targets: Sequence) -> None:
        """Stage the next step's HOST batches (numpy or pinned CPU tensors) on the
        copy stream; a following run_step with the same buffers consumes them
        (double-buffered H2D overlapping the current step's compute)."""
        n = len(batches)
        if len(targets) != n:
            raise UsageError(f"prefetch: expected {n} batches and targets, got {n} / {len(targets)}")
        self._check_inputs(batches, targets, "prefetch")
        if any(_on_device(x) for x in list(batches) + list(targets)):
            raise UsageError("prefetch: stages host buffers only")
        bp = (C.c_void_p * n)(*[_ptr(x) for x in batches])
        tp = (C.c_void_p * n)(*[_ptr(t) for t in targets])
        _check(lib.hp_cluster_prefetch(self._h, bp, tp))

    def trace(self) -> List[TraceEvent]:
        ev = (HpTraceEvent * 512)()
        k = lib.hp_cluster_trace(self._h, ev, 512)
        return [TraceEvent(Phase(e.phase), e.sub_batch, e.worker, e.bytes_total, e.bytes_max_sender)
                for e in ev[:k]]

    def worker_bytes(self, i: int):
        s = (C.c_int64 * 4)()
        r = (C.c_int64 * 4)()
        _check(lib.hp_cluster_worker_bytes(self._h, i, s, r))
        return list(s), list(r)

    def param(self, worker: int, which: int, layer: int) -> np.ndarray:
        """which: 0 conv kernels [F][C][R][S], 1 conv bias, 2 fc shard [in][out_i], 3 fc bias;
        +4 momentum. Reference layouts (WorkerState, cluster.hpp:77-84)."""
        n = lib.hp_cluster_param_size(self._h, worker, which, layer)
        if n < 0:
            raise UsageError("param: bad worker/which/layer")
        out = np.empty(n, dtype=np.float32)
        _check(lib.hp_cluster_read_param(self._h, worker, which, layer, out.ctypes.data, n))
        return out

    def decisions(self, worker: int, kind: int, layer: int) -> np.ndarray:
        """The last step's discrete forward decisions (parity tests): kind 0 conv
        ReLU mask uint8 [b*F*OH*OW], 1 conv pool argmax int32 (plane index h*OW+w),
        2 fc ReLU mask uint8 [n*out] with layer = turn * n_fc + fc layer (earlier
        turns need set_debug_capture(True)). See hp_cluster_debug_decisions."""
        n = lib.hp_cluster_debug_decisions(self._h, worker, kind, layer, None, 0)
        if n < 0:
            _check(4)
        out = np.empty(n, dtype=np.int32 if kind == 1 else np.uint8)
        if lib.hp_cluster_debug_decisions(self._h, worker, kind, layer, out.ctypes.data, n) < 0:
            _check(4)
        return out

    def set_debug_capture(self, on: bool) -> None:
        """Keep every turn's fc ReLU masks for decisions() (no graph replay while on)."""
        _check(lib.hp_cluster_set_debug_capture(self._h, int(bool(on))))

    def write_param(self, worker: int, which: int, layer: int, values) -> None:
        v = np.ascontiguousarray(values, dtype=np.float32).ravel()
        _check(lib.hp_cluster_write_param(self._h, worker, which, layer, v.ctypes.data, v.size))

    def gathered_model(self):
        """Cluster::gathered_model (cluster.cpp:417-437): (conv [(k, b)], fc [(w [in][out], b)])."""
        sp = self.spec
        ck = [np.empty(l.out_channels * l.in_channels * l.kernel * l.kernel, np.float32) for l in sp.conv_layers]
        cb = [np.empty(l.out_channels, np.float32) for l in sp.conv_layers]
        fw = [np.empty(l.in_dim * l.out_dim, np.float32) for l in sp.fc_layers]
        fb = [np.empty(l.out_dim, np.float32) for l in sp.fc_layers]
        arr = lambda xs: (C.c_void_p * len(xs))(*[x.ctypes.data for x in xs])
        _check(lib.hp_cluster_gather_model(self._h, arr(ck), arr(cb), arr(fw), arr(fb)))
        conv = [(k.reshape(l.out_channels, l.in_channels, l.kernel, l.kernel), b)
                for k, b, l in zip(ck, cb, sp.conv_layers)]
        fc = [(w.reshape(l.in_dim, l.out_dim), b) for w, b, l in zip(fw, fb, sp.fc_layers)]
        return conv, fc

    def set_skip_sync_broadcast(self, v: bool) -> None:
        _check(lib.hp_cluster_set_skip_sync_broadcast(self._h, int(bool(v))))

    def last_step_ms(self) -> float:
        return lib.hp_cluster_last_step_ms(self._h)

    def last_step_launches(self) -> int:
        return lib.hp_cluster_last_step_launches(self._h)

    def stream_ptr(self) -> int:
        """cudaStream_t every kernel of this cluster runs on (for CUDA-event timing)."""
        return lib.hp_cluster_stream(self._h) or 0

    def last_step_io(self):
        h2d, d2h = C.c_int64(), C.c_int64()
        lib.hp_cluster_last_step_io(self._h, C.byref(h2d), C.byref(d2h))
        return h2d.value, d2h.value

    def last_gemm_flops(self) -> float:
        return lib.hp_cluster_last_gemm_flops(self._h)

    def set_graphs(self, on: bool) -> None:
        """Replay steps as captured CUDA graphs (default on; see hp_cluster_set_graphs)."""
        _check(lib.hp_cluster_set_graphs(self._h, int(bool(on))))

    def set_fuse_fc_sgd(self, on: bool) -> None:
        """FC weight update in the wgrad GEMM epilogue (default on)."""
        _check(lib.hp_cluster_set_fuse_fc_sgd(self._h, int(bool(on))))

    def set_shift_conv(self, on: bool) -> None:
        """bf16 stride-1 convs via the flat-shift kernel (default on) or TMA im2col."""
        _check(lib.hp_cluster_set_shift_conv(self._h, int(bool(on))))

    def set_profile(self, on: bool) -> None:
        _check(lib.hp_cluster_set_profile(self._h, int(bool(on))))

    def marker_graph(self, batches: Sequence, targets: Sequence, hp: HyperParams, lr: Optional[float] = None):
        """Debug: (tags, reach) of one captured-but-not-run step; reach[i][k] is
        True when marker tags[k] is reachable from tags[i] in the step graph
        (see hp_cluster_debug_marker_graph for the tag scheme)."""
        lr = hp.lr if lr is None else lr
        n = len(batches)
        self._check_inputs(batches, targets, "marker_graph")
        device = _on_device(batches[0])
        bp = (C.c_void_p * n)(*[_ptr(x) for x in batches])
        tp = (C.c_void_p * n)(*[_ptr(t) for t in targets])
        h = HpHyper(hp.momentum, hp.lr, hp.weight_decay, 0 if hp.fc_partial_lr is None else 1,
                    0.0 if hp.fc_partial_lr is None else hp.fc_partial_lr)
        cap = 1024
        tags = (C.c_int32 * cap)()
        reach = (C.c_uint8 * (cap * cap))()
        nm = C.c_int()
        _check(lib.hp_cluster_debug_marker_graph(self._h, bp, tp, 1 if device else 0, C.byref(h), lr, tags,
                                                 reach, cap, C.byref(nm)))
        m = nm.value
        r = np.frombuffer(reach, dtype=np.uint8, count=m * m).reshape(m, m).astype(bool)
        return list(tags[:m]), r

    def gemm_profile(self):
        """[(tag, layer, flops, ms)] for the last profiled step, launch order."""
        buf = (HpGemmProf * 4096)()
        k = lib.hp_cluster_gemm_profile(self._h, buf, 4096)
        return [(e.tag.decode(), e.layer, e.flops, e.ms) for e in buf[:k]]


# ---------------------------------------------------------------- host helpers
def step_accounting(spec: ModelSpec, config: ClusterConfig, steps: int = 1):
    """Analytic byte counters and trace (cluster.cpp:466-673) without a GPU:
    (bytes_sent[4], trace, [(sent[4], received[4]) per worker])."""
    sc, keep = _spec_c(spec)
    cfg = HpClusterConfig()
    cfg.workers, cfg.per_worker_batch = config.workers, config.per_worker_batch
    cfg.scheme, cfg.variable_batch = int(config.scheme), int(bool(config.variable_batch))
    cfg.precision, cfg.seed, cfg.math_mode = int(config.precision), config.seed, int(config.math_mode)
    bs = (C.c_int64 * 4)()
    tr = (HpTraceEvent * 512)()
    ne = C.c_int()
    K = config.workers
    ws, wr = (C.c_int64 * (4 * K))(), (C.c_int64 * (4 * K))()
    _check(lib.hp_step_accounting(C.byref(sc), C.byref(cfg), steps, bs, tr, 512, C.byref(ne), ws, wr))
    trace = [(e.phase, e.sub_batch, e.worker, e.bytes_total, e.bytes_max_sender) for e in tr[:ne.value]]
    per = [(list(ws[4 * w:4 * w + 4]), list(wr[4 * w:4 * w + 4])) for w in range(K)]
    return list(bs), trace, per



def shard_range(total: int, parts: int, idx: int):
    b, e = C.c_int64(), C.c_int64()
    lib.hp_shard_range(total, parts, idx, C.byref(b), C.byref(e))
    return b.value, e.value


def gaussian(seed: int, n: int) -> np.ndarray:
    """GaussianSampler(seed).next() x n (rng.hpp:26-56), host replay."""
    out = np.empty(n, dtype=np.float64)
    lib.hp_gaussian_fill(seed, out.ctypes.data_as(C.POINTER(C.c_double)), n)
    return out


def gaussian_f32(seed: int, n: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    lib.hp_gaussian_fill_f32(seed, scale, out.ctypes.data_as(C.POINTER(C.c_float)), n)
    return out
