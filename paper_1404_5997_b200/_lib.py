"""ctypes binding of the C ABI in include/hpsim_b200.h.

The shared library is built in-tree (paper_1404_5997_b200/lib/libhpsim_b200.so).
There is no fallback: if the library is missing or fails to load, importing
the package raises, so no test or benchmark can silently run without the
CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HP_DEV_LIB") or os.path.join(_HERE, "lib", "libhpsim_b200.so")  # HP_DEV_LIB: dev variant builds


class HpConvLayer(C.Structure):
    _fields_ = [
        ("in_channels", C.c_int64),
        ("out_channels", C.c_int64),
        ("kernel", C.c_int32),
        ("stride", C.c_int32),
        ("pad", C.c_int32),
        ("relu", C.c_int32),
        ("floor_mode", C.c_int32),
        ("lrn_size", C.c_int32),
        ("lrn_alpha", C.c_double),
        ("lrn_beta", C.c_double),
        ("lrn_k", C.c_double),
        ("pool_kernel", C.c_int32),
        ("pool_stride", C.c_int32),
    ]


class HpFcLayer(C.Structure):
    _fields_ = [("in_dim", C.c_int64), ("out_dim", C.c_int64), ("relu", C.c_int32)]


class HpModelSpec(C.Structure):
    _fields_ = [
        ("conv", C.POINTER(HpConvLayer)),
        ("n_conv", C.c_int32),
        ("fc", C.POINTER(HpFcLayer)),
        ("n_fc", C.c_int32),
        ("input_shape", C.c_int64 * 3),
        ("num_classes", C.c_int64),
    ]


class HpClusterConfig(C.Structure):
    _fields_ = [
        ("workers", C.c_int32),
        ("per_worker_batch", C.c_int64),
        ("scheme", C.c_int32),
        ("variable_batch", C.c_int32),
        ("precision", C.c_int32),
        ("seed", C.c_uint64),
        ("math_mode", C.c_int32),
        ("transport", C.c_int32),
        ("rank", C.c_int32),
        ("device", C.c_int32),
        ("nccl_id", C.c_ubyte * 128),
    ]


class HpHyper(C.Structure):
    _fields_ = [
        ("momentum", C.c_double),
        ("lr", C.c_double),
        ("weight_decay", C.c_double),
        ("has_fc_partial_lr", C.c_int32),
        ("fc_partial_lr", C.c_double),
    ]


class HpTraceEvent(C.Structure):
    _fields_ = [
        ("phase", C.c_int32),
        ("sub_batch", C.c_int32),
        ("worker", C.c_int32),
        ("bytes_total", C.c_int64),
        ("bytes_max_sender", C.c_int64),
    ]


class HpStepMetrics(C.Structure):
    _fields_ = [
        ("loss", C.c_double),
        ("fc_update_count", C.c_int32),
        ("conv_update_count", C.c_int32),
        ("bytes_sent", C.c_int64 * 4),
        ("n_events", C.c_int32),
    ]


class HpGemmProf(C.Structure):
    _fields_ = [("tag", C.c_char * 16), ("layer", C.c_int32), ("flops", C.c_double), ("ms", C.c_double)]


class HpGemmDesc(C.Structure):
    _fields_ = [
        ("math", C.c_int32),
        ("a", C.c_void_p), ("a_mn", C.c_int32), ("lda", C.c_int64),
        ("b", C.c_void_p), ("b_mn", C.c_int32), ("ldb", C.c_int64),
        ("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32),
        ("c", C.c_void_p), ("ldc", C.c_int64), ("c_type", C.c_int32), ("c_trans", C.c_int32),
        ("alpha", C.c_float), ("beta", C.c_int32),
        ("bias", C.c_void_p), ("bias_mode", C.c_int32), ("relu", C.c_int32),
        ("mask", C.c_void_p), ("ldmask", C.c_int64), ("mask_type", C.c_int32),
        ("mask_trans", C.c_int32),
        ("splits", C.c_int32), ("bn", C.c_int32),
        ("ws", C.c_void_p),
        ("cta2", C.c_int32),
    ]


class HpDatasetSpec(C.Structure):
    _fields_ = [("num_examples", C.c_int64), ("channels", C.c_int32), ("height", C.c_int32),
                ("width", C.c_int32), ("num_classes", C.c_int32), ("seed", C.c_uint64), ("separation", C.c_double)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P = C.c_void_p
    sigs = {
        "hp_last_error": ([], C.c_char_p),
        "hp_version": ([], C.c_char_p),
        "hp_shard_range": ([C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], None),
        "hp_gaussian_fill": ([C.c_uint64, C.POINTER(C.c_double), C.c_int64], None),
        "hp_gaussian_fill_f32": ([C.c_uint64, C.c_double, C.POINTER(C.c_float), C.c_int64], None),
        "hp_kernel_gemm": ([C.POINTER(HpGemmDesc), P], C.c_int),
        "hp_kernel_conv_shift": ([P, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int, P, C.c_int, P],
                                 C.c_int),
        "hp_kernel_gemm_splits": ([C.POINTER(HpGemmDesc)], C.c_int),
        "hp_debug_gemm_force": ([C.c_int, C.c_int], None),
        "hp_debug_gemm_flags": ([C.c_int], None),
        "hp_kernel_conv_fprop": ([C.c_int, P, C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int, C.c_int,
                                  C.c_int, C.c_int, C.c_int, P, P], C.c_int),
        "hp_kernel_conv_wgrad": ([C.c_int, P, C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int, C.c_int,
                                  C.c_int, C.c_int, C.c_int, P, P, C.c_int64, P], C.c_int),
        "hp_kernel_lrn_pool_fwd": ([C.c_int, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float,
                                    C.c_float, C.c_float, C.c_int, C.c_int, P, P, P], C.c_int),
        "hp_kernel_lrn_pool_bwd": ([C.c_int, P, P, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float,
                                    C.c_float, C.c_float, C.c_int, C.c_int, C.c_int, P, P, P], C.c_int),
        "hp_kernel_sgd": ([P, P, P, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_float, C.c_int, P, P],
                          C.c_int),
        "hp_kernel_conv_dgrad": ([C.c_int, P, C.c_int, C.c_int, C.c_int, C.c_int, P, C.c_int, C.c_int,
                                  C.c_int, C.c_int, P, P], C.c_int),
        "hp_data_generate": ([C.POINTER(HpDatasetSpec), C.c_int64, C.c_int64, P, P, C.c_int, P], C.c_int),
        "hp_data_class_of": ([C.POINTER(HpDatasetSpec), C.c_int64, C.POINTER(C.c_int64)], C.c_int),
    }
    optional = {
        "hp_cluster_create": ([C.POINTER(HpModelSpec), C.POINTER(HpClusterConfig), C.POINTER(P)], C.c_int),
        "hp_cluster_destroy": ([P], None),
        "hp_nccl_unique_id": ([C.POINTER(C.c_ubyte * 128)], C.c_int),
        "hp_cluster_prefetch": ([P, P, P], C.c_int),
        "hp_cluster_run_step": ([P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int,
                                 C.POINTER(HpHyper), C.c_double, C.POINTER(HpStepMetrics)], C.c_int),
        "hp_cluster_trace": ([P, C.POINTER(HpTraceEvent), C.c_int], C.c_int),
        "hp_cluster_worker_bytes": ([P, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
        "hp_cluster_param_size": ([P, C.c_int, C.c_int, C.c_int], C.c_int64),
        "hp_cluster_read_param": ([P, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64], C.c_int),
        "hp_cluster_write_param": ([P, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64], C.c_int),
        "hp_cluster_debug_decisions": ([P, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int64], C.c_int64),
        "hp_cluster_set_debug_capture": ([P, C.c_int], C.c_int),
        "hp_cluster_gather_model": ([P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                     C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)], C.c_int),
        "hp_cluster_set_skip_sync_broadcast": ([P, C.c_int], C.c_int),
        "hp_cluster_last_step_ms": ([P], C.c_double),
        "hp_cluster_last_step_launches": ([P], C.c_int64),
        "hp_cluster_stream": ([P], C.c_void_p),
        "hp_step_accounting": ([C.POINTER(HpModelSpec), C.POINTER(HpClusterConfig), C.c_int,
                                C.POINTER(C.c_int64), C.POINTER(HpTraceEvent), C.c_int, C.POINTER(C.c_int),
                                C.POINTER(C.c_int64), C.POINTER(C.c_int64)], C.c_int),
        "hp_cluster_last_step_io": ([P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)], None),
        "hp_cluster_last_gemm_flops": ([P], C.c_double),
        "hp_cluster_set_profile": ([P, C.c_int], C.c_int),
        "hp_cluster_set_fuse_fc_sgd": ([P, C.c_int], C.c_int),
        "hp_cluster_set_shift_conv": ([P, C.c_int], C.c_int),
        "hp_cluster_set_graphs": ([P, C.c_int], C.c_int),
        "hp_cluster_gemm_profile": ([P, C.POINTER(HpGemmProf), C.c_int], C.c_int),
        "hp_cluster_debug_marker_graph": ([P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.c_int,
                                           C.POINTER(HpHyper), C.c_double, C.POINTER(C.c_int32),
                                           C.POINTER(C.c_uint8), C.c_int, C.POINTER(C.c_int)], C.c_int),
    }
    for name, (args, res) in list(sigs.items()) + list(optional.items()):
        fn = getattr(lib, name, None)
        if fn is None:
            if name in sigs:
                raise ImportError(f"{LIB_PATH} does not export {name}")
            continue
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def last_error() -> str:
    return lib.hp_last_error().decode()
