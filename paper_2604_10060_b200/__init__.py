"""B200-native cluster-level KV-cache hot path (Mosaic, arXiv 2604.10060).

The product is `_lib/libkvc.so` (C++ host control plane + sm_100a kernels behind the C-ABI of
include/kvc.h); `api.ClusterKVCache` is the Python mirror of the reference's StreamEngine-level
interface over that ABI.
"""
from .api import (CAUSES, DTYPE_BF16, DTYPE_F32, ClusterKVCache, Config, KvcError, LayerMeta,
                  lib)

__all__ = ["ClusterKVCache", "Config", "KvcError", "LayerMeta", "lib", "CAUSES", "DTYPE_F32",
           "DTYPE_BF16"]
