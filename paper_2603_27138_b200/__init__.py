"""B200-native ScoutAttention decode hot path (arxiv 2603.27138).

The product is libscout_b200.so (sm_100a kernels + C ABI, include/scout_b200.h).
`ops` drives it on torch device tensors (tests, bench); `engine` wraps the C++
decode-step engine (csrc/engine.cpp) and `tier` the device-resident
TieredKvCache (K5); `sharding` splits requests across ranks. The reference's
C++ hot-path API (select_topk, partial_attention, merge, finalize, build_digest,
digest_score) is restated on the C ABI by the header-only include/scout_b200.hpp.
Importing this package does not touch the GPU.
"""
from ._capi import LIB_PATH, ScoutError, lib  # noqa: F401

HEAD_DIM = 128
BLOCK_SIZE = 64
