"""rserve-b200: B200-native implementation of RServe's intra-request pipeline.

Chunked multimodal encoding (Algorithm 1) -> device embedding tracker ->
chunked pipeline-parallel prefill, with the reference's (arxiv 2509.24381,
``lmmsim``) request / tracker / scheduler API kept intact. The host side is
C++ (include/lmmsim/, paper_2509_24381_b200/csrc/host/); kernels are
hand-written sm_100a CUDA (tcgen05/TMEM/TMA GEMM, flash attention, tracker
data plane). Python is a thin ctypes layer over the C-ABI in include/rserve.h.
"""
from . import _native  # noqa: F401  (raises ImportError when the .so is missing)
from ._native import (AlignmentError, ConfigError, DataError, DependencyViolation,  # noqa: F401
                      DeviceError, DoubleEncodeError, InputError, InternalError, IoError,
                      RegistryError, SimError, version)

__all__ = ["version", "SimError", "ConfigError", "RegistryError", "DoubleEncodeError",
           "AlignmentError", "DependencyViolation", "InputError", "DataError", "IoError",
           "InternalError", "DeviceError"]
