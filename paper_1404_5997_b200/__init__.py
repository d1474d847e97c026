"""paper_1404_5997_b200 — B200-native hybrid data/model-parallel CNN training
step ("One weird trick", arXiv:1404.5997) behind the reference's hpsim
Cluster interface. The compute path is libhpsim_b200.so (CUDA sm_100a,
tcgen05 GEMMs, NCCL); importing this package fails if it is missing.
"""
from ._lib import LIB_PATH, lib  # noqa: F401  (raises ImportError when the .so is absent)
from .api import (Cluster, ClusterConfig, ConfigError, ConvLayerSpec, CudaError, DimensionError,  # noqa: F401
                  DomainError, FcLayerSpec, HpsimError, HyperParams, MathMode, ModelSpec, MsgClass, NcclError,
                  Phase, Precision, Scheme, StepMetrics, StepResult, TraceEvent, Transport, UsageError,
                  gaussian, gaussian_f32, nccl_unique_id, shard_range, step_accounting)
from .specs import alexnet_1col, alexnet_standin_227, synthetic_batch, tiny_cnn  # noqa: F401
from . import data  # noqa: F401  (input pipeline: SPEC data_gen on the GPU)

__version__ = "0.1.0"
