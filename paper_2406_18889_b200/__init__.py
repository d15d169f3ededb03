"""B200-native tensor-network random-circuit sampler (arXiv 2406.18889 hot path).

The product is the native library ``_native/libpaper_2406_18889_b200.so``
(host C++ + sm_100a CUDA kernels behind the C ABI in ``include/rcsg.h``);
this package is its Python binding (``api``) and the multi-GPU slice
scheduler (``scheduler``).
"""
from .api import (CapacityError, ConfigError, DeviceError, NumericFault, Problem,  # noqa: F401
                  build_candidate_set, broken_configs, direct_sample, execute_desc, lexkey,
                  member, split_next, top_k_select, xeb)

__all__ = ["Problem", "ConfigError", "NumericFault", "CapacityError", "DeviceError",
           "build_candidate_set", "top_k_select", "direct_sample", "xeb", "member", "lexkey",
           "split_next", "broken_configs", "execute_desc"]
