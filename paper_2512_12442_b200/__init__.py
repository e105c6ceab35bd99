"""paper_2512_12442_b200 -- B200-native LCP hot path of arxiv 2512.12442.

The product is `liblcp.so` (sm_100a kernels behind the C ABI of
`include/lcp.h`); `lcp.py` is its ctypes binding, `dist.py` the z-slab
multi-GPU driver over torch.distributed.  Nothing here imports `oracle/`.
"""
from .lcp import (Context, LcpError, EXPORTS, K_SE, K_MATERN52, FP32, FP64, NODE_DTYPE,  # noqa: F401
                  config_args, load_library, LIB_PATH)
