"""B200-native ScoutAttention decode hot path (arxiv 2603.27138).

The product is libscout_b200.so (sm_100a kernels + C ABI, include/scout_b200.h).
`ops` drives it on torch device tensors; `reference_api` restates the
reference's C++ hot-path API (select_topk, partial_attention, merge, finalize,
build_digest, digest_score) on top of it; `engine` is the host-side decode-step
orchestration. Importing this package does not touch the GPU.
"""
from ._capi import LIB_PATH, ScoutError, lib  # noqa: F401

HEAD_DIM = 128
BLOCK_SIZE = 64
