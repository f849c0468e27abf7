"""B200-native LANCE: int8 Winograd-domain convolution (arXiv 2003.08646).

The reference's ``lance_gemm`` path (engines.hpp:492-536) rebuilt as four
hand-written sm_100a kernels behind a C ABI (include/lance_b200.h), with the
reference's operator API mirrored here and in include/lance/b200.hpp.
"""
from .api import (ConvSpec, Granularity, LanceConfig, LanceConv, LanceDeviceError,
                  LanceError, LanceMode, LanceNaNError, QuantParams, direct_multiply_count,
                  lance_gemm, params_array, uniform_floats, validate,
                  winograd_multiply_count, winograd_multiply_count_tiled)

__all__ = ["ConvSpec", "Granularity", "LanceConfig", "LanceConv", "LanceDeviceError",
           "LanceError", "LanceMode", "LanceNaNError", "QuantParams",
           "direct_multiply_count", "lance_gemm", "params_array", "uniform_floats",
           "validate", "winograd_multiply_count", "winograd_multiply_count_tiled"]
