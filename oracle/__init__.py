"""Oracle bindings — TEST INFRASTRUCTURE ONLY.

Two checkers live here, both CPU-only:

* ``Oracle*``: the plain-C restatement in oracle/hpsim_oracle.c (double
  precision, reference loop orders, plus the AlexNet superset: floor-mode
  geometry, LRN, overlapping max-pool).
* ``Ref*``: the unmodified reference (/root/reference/proj/core) compiled by
  ``make -C oracle ref`` into oracle/_ref/libhpsim_ref.so (gitignored; it
  travels to the GPU box as a built artefact). Absent -> ``ref_available()``
  is False and tests fall back to tests/golden/ fixtures.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package. The product (paper_1404_5997_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "build", "libhpsim_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libhpsim_ref.so")


class ConvLayer(C.Structure):
    _fields_ = [
        ("in_channels", C.c_int64), ("out_channels", C.c_int64),
        ("kernel", C.c_int32), ("stride", C.c_int32), ("pad", C.c_int32), ("relu", C.c_int32),
        ("floor_mode", C.c_int32), ("lrn_size", C.c_int32),
        ("lrn_alpha", C.c_double), ("lrn_beta", C.c_double), ("lrn_k", C.c_double),
        ("pool_kernel", C.c_int32), ("pool_stride", C.c_int32),
    ]


class FcLayer(C.Structure):
    _fields_ = [("in_dim", C.c_int64), ("out_dim", C.c_int64), ("relu", C.c_int32)]


class ModelSpecC(C.Structure):
    _fields_ = [
        ("conv", C.POINTER(ConvLayer)), ("n_conv", C.c_int32),
        ("fc", C.POINTER(FcLayer)), ("n_fc", C.c_int32),
        ("input_shape", C.c_int64 * 3), ("num_classes", C.c_int64),
    ]


class ClusterConfigC(C.Structure):
    _fields_ = [
        ("workers", C.c_int32), ("per_worker_batch", C.c_int64), ("scheme", C.c_int32),
        ("variable_batch", C.c_int32), ("precision", C.c_int32), ("seed", C.c_uint64),
    ]


class HyperC(C.Structure):
    _fields_ = [
        ("momentum", C.c_double), ("lr", C.c_double), ("weight_decay", C.c_double),
        ("has_fc_partial_lr", C.c_int32), ("fc_partial_lr", C.c_double),
    ]


class TraceEventC(C.Structure):
    _fields_ = [
        ("phase", C.c_int32), ("sub_batch", C.c_int32), ("worker", C.c_int32),
        ("bytes_total", C.c_int64), ("bytes_max_sender", C.c_int64),
    ]


class StepMetricsC(C.Structure):
    _fields_ = [
        ("loss", C.c_double), ("fc_update_count", C.c_int32), ("conv_update_count", C.c_int32),
        ("bytes_sent", C.c_int64 * 4), ("n_events", C.c_int32),
    ]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


SCHEMES = {"A": 0, "B": 1, "C": 2, "a": 0, "b": 1, "c": 2, 0: 0, 1: 1, 2: 2}

_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _load_oracle() -> C.CDLL:
    if not os.path.exists(ORACLE_LIB):
        raise ImportError(f"{ORACLE_LIB} missing: run `make -C oracle`")
    lib = C.CDLL(ORACLE_LIB)
    P = C.c_void_p
    lib.or_last_error.restype = C.c_char_p
    lib.or_validate.argtypes = [C.POINTER(ModelSpecC)]
    lib.or_flattened_conv_size.argtypes = [C.POINTER(ModelSpecC)]
    lib.or_flattened_conv_size.restype = C.c_int64
    lib.or_conv_output_sizes.argtypes = [C.POINTER(ModelSpecC), _I64]
    lib.or_cluster_create.argtypes = [C.POINTER(ModelSpecC), C.POINTER(ClusterConfigC), C.POINTER(C.c_int)]
    lib.or_cluster_create.restype = P
    lib.or_cluster_destroy.argtypes = [P]
    lib.or_cluster_run_step.argtypes = [P, C.POINTER(_D), C.POINTER(_D), C.POINTER(HyperC), C.c_double,
                                        C.POINTER(StepMetricsC)]
    lib.or_cluster_trace.argtypes = [P, C.POINTER(TraceEventC), C.c_int]
    lib.or_cluster_worker_bytes.argtypes = [P, C.c_int, _I64, _I64]
    lib.or_cluster_param_size.argtypes = [P, C.c_int, C.c_int, C.c_int]
    lib.or_cluster_param_size.restype = C.c_int64
    lib.or_cluster_read_param.argtypes = [P, C.c_int, C.c_int, C.c_int, _D, C.c_int64]
    lib.or_cluster_write_param.argtypes = [P, C.c_int, C.c_int, C.c_int, _D, C.c_int64]
    lib.or_cluster_set_skip_sync_broadcast.argtypes = [P, C.c_int]
    lib.or_cluster_set_storage_rounding.argtypes = [P, C.c_int]
    lib.or_cluster_force_decisions.argtypes = [P, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64]
    lib.or_cluster_decision_stats.argtypes = [P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                              C.POINTER(C.c_double)]
    lib.or_set_threads.argtypes = [C.c_int]
    lib.or_gaussian_fill.argtypes = [C.c_uint64, _D, C.c_int64]
    lib.or_uniform_u64.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.c_int64]
    i64 = C.c_int64
    lib.or_conv2d_forward.argtypes = [_D, i64, i64, i64, i64, _D, i64, i64, i64, C.c_int, C.c_int, C.c_int, _D]
    lib.or_conv2d_backward.argtypes = [_D, i64, i64, i64, i64, _D, i64, i64, i64, C.c_int, C.c_int, C.c_int,
                                       _D, _D, _D]
    for n in ("or_matmul", "or_matmul_tn", "or_matmul_nt"):
        getattr(lib, n).argtypes = [_D, _D, _D, i64, i64, i64]
    lib.or_logistic_xent.argtypes = [_D, _D, i64, i64, _D, _D]
    lib.or_momentum_update.argtypes = [_D, _D, _D, i64, C.c_double, C.c_double, C.c_double]
    F = C.POINTER(C.c_float)
    lib.or_momentum_update_f32.argtypes = [F, F, F, i64, C.c_double, C.c_double, C.c_double]
    lib.or_maxpool_forward.argtypes = [_D, i64, i64, i64, i64, C.c_int, C.c_int, _D, C.POINTER(C.c_int32)]
    lib.or_maxpool_backward.argtypes = [_D, C.POINTER(C.c_int32), i64, i64, i64, i64, C.c_int, C.c_int, _D]
    lib.or_lrn_forward.argtypes = [_D, i64, i64, i64, C.c_int, C.c_double, C.c_double, C.c_double, _D, _D]
    lib.or_lrn_backward.argtypes = [_D, _D, _D, i64, i64, i64, C.c_int, C.c_double, C.c_double, _D]
    return lib


_oracle: Optional[C.CDLL] = None
_ref: Optional[C.CDLL] = None


def oracle_lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        _oracle = _load_oracle()
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        if not ref_available():
            raise ImportError(f"{REF_LIB} missing: run `make -C oracle ref` where /root/reference exists")
        lib = C.CDLL(REF_LIB)
        P = C.c_void_p
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_cluster_create.argtypes = [C.POINTER(ModelSpecC), C.POINTER(ClusterConfigC), C.POINTER(C.c_int)]
        lib.ref_cluster_create.restype = P
        lib.ref_cluster_destroy.argtypes = [P]
        lib.ref_cluster_set_skip_sync_broadcast.argtypes = [P, C.c_int]
        lib.ref_cluster_run_step.argtypes = [P, C.POINTER(_D), C.POINTER(_D), C.POINTER(HyperC), C.c_double,
                                             C.POINTER(StepMetricsC)]
        lib.ref_cluster_trace.argtypes = [P, C.POINTER(TraceEventC), C.c_int]
        lib.ref_cluster_worker_bytes.argtypes = [P, C.c_int, _I64, _I64]
        lib.ref_cluster_param_size.argtypes = [P, C.c_int, C.c_int, C.c_int]
        lib.ref_cluster_param_size.restype = C.c_int64
        lib.ref_cluster_read_param.argtypes = [P, C.c_int, C.c_int, C.c_int, _D, C.c_int64]
        lib.ref_cluster_write_param.argtypes = [P, C.c_int, C.c_int, C.c_int, _D, C.c_int64]
        lib.ref_gaussian_fill.argtypes = [C.c_uint64, _D, C.c_int64]
        lib.ref_count_stats.argtypes = [C.POINTER(ModelSpecC), _I64]
        i64 = C.c_int64
        lib.ref_conv2d_forward.argtypes = [C.c_int, _D, i64, i64, i64, i64, _D, i64, i64, i64, C.c_int, C.c_int, _D]
        lib.ref_conv2d_backward.argtypes = [C.c_int, _D, i64, i64, i64, i64, _D, i64, i64, i64, C.c_int, C.c_int,
                                            _D, i64, i64, _D, _D]
        lib.ref_matmul.argtypes = [C.c_int, C.c_int, _D, _D, _D, i64, i64, i64, i64]
        lib.ref_logistic_xent.argtypes = [C.c_int, _D, _D, i64, i64, _D, _D]
        lib.ref_momentum_update.argtypes = [C.c_int, _D, _D, _D, i64, C.c_double, C.c_double, C.c_double]
        lib.ref_lr_at.argtypes = [C.c_double, C.c_double, C.POINTER(C.c_int)]
        lib.ref_lr_at.restype = C.c_double
        lib.ref_single_create.argtypes = [C.POINTER(ModelSpecC), C.c_uint64, C.c_int, C.POINTER(C.c_int)]
        lib.ref_single_create.restype = P
        lib.ref_single_destroy.argtypes = [P]
        lib.ref_single_step.argtypes = [P, _D, _D, i64, C.POINTER(HyperC), C.c_double, _D]
        lib.ref_single_read.argtypes = [P, C.c_int, C.c_int, _D, i64]
        _ref = lib
    return _ref


# ------------------------------------------------------------------ specs

def make_spec_c(spec) -> ModelSpecC:
    """Duck-typed: ``spec`` has conv_layers / fc_layers / input_shape / num_classes
    with the hpsim field names (model.hpp:24-49) and the optional superset fields."""
    convs = (ConvLayer * max(1, len(spec.conv_layers)))()
    for i, l in enumerate(spec.conv_layers):
        convs[i] = ConvLayer(
            l.in_channels, l.out_channels, l.kernel, l.stride, l.pad, int(bool(l.relu)),
            int(bool(getattr(l, "floor_mode", False))), int(getattr(l, "lrn_size", 0)),
            float(getattr(l, "lrn_alpha", 0.0)), float(getattr(l, "lrn_beta", 0.0)),
            float(getattr(l, "lrn_k", 0.0)), int(getattr(l, "pool_kernel", 0)),
            int(getattr(l, "pool_stride", 0)))
    fcs = (FcLayer * max(1, len(spec.fc_layers)))()
    for i, l in enumerate(spec.fc_layers):
        fcs[i] = FcLayer(l.in_dim, l.out_dim, int(bool(l.relu)))
    s = ModelSpecC()
    s.conv = C.cast(convs, C.POINTER(ConvLayer))
    s.n_conv = len(spec.conv_layers)
    s.fc = C.cast(fcs, C.POINTER(FcLayer))
    s.n_fc = len(spec.fc_layers)
    for i in range(3):
        s.input_shape[i] = int(spec.input_shape[i])
    s.num_classes = int(spec.num_classes)
    s._keep = (convs, fcs)  # keep arrays alive
    return s


def make_hyper_c(momentum=0.9, lr=0.01, weight_decay=0.0, fc_partial_lr=None) -> HyperC:
    h = HyperC()
    h.momentum, h.lr, h.weight_decay = momentum, lr, weight_decay
    h.has_fc_partial_lr = 0 if fc_partial_lr is None else 1
    h.fc_partial_lr = 0.0 if fc_partial_lr is None else float(fc_partial_lr)
    return h


def _ptr_array(arrs: Sequence[np.ndarray]):
    arr = (_D * len(arrs))()
    for i, a in enumerate(arrs):
        arr[i] = _dp(a)
    return arr


class _ClusterBase:
    """Common driver over the restatement (or_*) and the reference (ref_*)."""

    prefix = "or_"

    def __init__(self, spec, workers=1, per_worker_batch=128, scheme="B", variable_batch=False,
                 precision="double", seed=0):
        self.lib = self._lib()
        self.spec = spec
        self.spec_c = make_spec_c(spec)
        cfg = ClusterConfigC()
        cfg.workers = workers
        cfg.per_worker_batch = per_worker_batch
        cfg.scheme = SCHEMES[scheme]
        cfg.variable_batch = int(bool(variable_batch))
        cfg.precision = 0 if precision in ("single", 0) else 1
        cfg.seed = seed
        self.cfg = cfg
        st = C.c_int(0)
        self.h = self._fn("cluster_create")(C.byref(self.spec_c), C.byref(cfg), C.byref(st))
        if not self.h:
            raise OracleError(st.value, self._err())
        self.workers = workers
        self.b = per_worker_batch

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _err(self):
        return self._fn("last_error")().decode()

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._err())

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            self._fn("cluster_destroy")(h)
            self.h = None

    def run_step(self, batches: Sequence[np.ndarray], targets: Sequence[np.ndarray], hyper=None, lr=None):
        hyper = hyper or make_hyper_c()
        lr = hyper.lr if lr is None else lr
        xs = [np.ascontiguousarray(x, dtype=np.float64) for x in batches]
        ts = [np.ascontiguousarray(t, dtype=np.float64) for t in targets]
        m = StepMetricsC()
        self._check(self._fn("cluster_run_step")(self.h, _ptr_array(xs), _ptr_array(ts), C.byref(hyper), lr,
                                                 C.byref(m)))
        return m

    def trace(self):
        ev = (TraceEventC * 256)()
        n = self._fn("cluster_trace")(self.h, ev, 256)
        return [(e.phase, e.sub_batch, e.worker, e.bytes_total, e.bytes_max_sender) for e in ev[:n]]

    def worker_bytes(self, i):
        s = (C.c_int64 * 4)()
        r = (C.c_int64 * 4)()
        self._check(self._fn("cluster_worker_bytes")(self.h, i, s, r))
        return list(s), list(r)

    def param(self, worker, which, layer):
        n = self._fn("cluster_param_size")(self.h, worker, which, layer)
        if n < 0:
            raise OracleError(4, "bad param index")
        out = np.empty(n, dtype=np.float64)
        self._check(self._fn("cluster_read_param")(self.h, worker, which, layer, _dp(out), n))
        return out

    def write_param(self, worker, which, layer, values):
        v = np.ascontiguousarray(values, dtype=np.float64).ravel()
        self._check(self._fn("cluster_write_param")(self.h, worker, which, layer, _dp(v), v.size))

    def set_skip_sync_broadcast(self, v: bool):
        self._fn("cluster_set_skip_sync_broadcast")(self.h, int(bool(v)))

    def gathered_model(self):
        """cluster.cpp:417-437 assembled from worker params."""
        K = self.workers
        conv = [(self.param(0, 0, l), self.param(0, 1, l)) for l in range(len(self.spec.conv_layers))]
        fc = []
        for l, L in enumerate(self.spec.fc_layers):
            ws = [self.param(i, 2, l).reshape(L.in_dim, -1) for i in range(K)]
            bs = [self.param(i, 3, l) for i in range(K)]
            fc.append((np.concatenate(ws, axis=1), np.concatenate(bs)))
        return conv, fc


class OracleCluster(_ClusterBase):
    def set_storage_rounding(self, mode: str):
        """'double' (the reference restatement) or 'bf16' (round stored tensors
        where the B200 bf16 math mode stores them; see hpsim_oracle.c)."""
        self._check(self.lib.or_cluster_set_storage_rounding(self.h, {"double": 0, "bf16": 1}[mode]))

    def force_decisions(self, worker: int, kind: int, layer: int, values):
        """Replay these ReLU masks (kind 0 conv, 2 fc; uint8) / pool argmax
        (kind 1, int32 plane index) in the next step; None clears."""
        if values is None:
            self._check(self.lib.or_cluster_force_decisions(self.h, worker, kind, layer, None, 0))
            return
        v = np.ascontiguousarray(values, dtype=np.int32 if kind == 1 else np.uint8)
        self._check(self.lib.or_cluster_force_decisions(self.h, worker, kind, layer, v.ctypes.data, v.size))

    def decision_stats(self, worker: int, kind: int, layer: int):
        """(mismatches, max_gap) of the last step's forced decisions against the
        oracle's own: ReLU -- |z| / rms(z); pool -- relative value gap."""
        m, g = C.c_int64(0), C.c_double(0.0)
        self._check(self.lib.or_cluster_decision_stats(self.h, worker, kind, layer, C.byref(m), C.byref(g)))
        return m.value, g.value

    prefix = "or_"

    @staticmethod
    def _lib():
        return oracle_lib()


class RefCluster(_ClusterBase):
    prefix = "ref_"

    @staticmethod
    def _lib():
        return ref_lib()


def gaussian(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    oracle_lib().or_gaussian_fill(seed, _dp(out), n)
    return out


def uniform_u64(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    oracle_lib().or_uniform_u64(seed, out.ctypes.data_as(C.POINTER(C.c_uint64)), n)
    return out


def set_threads(n: int) -> None:
    oracle_lib().or_set_threads(n)
