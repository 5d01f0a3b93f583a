"""ctypes binding of the C ABI declared in include/scout_b200.h.

This is exactly the binding a maintainer of a Python caller would add (see
INTEGRATION.md); the product path loads libscout_b200.so and fails loudly if
it is missing — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("SCOUT_B200_LIB", Path(__file__).resolve().parent / "libscout_b200.so"))

SCOUT_OK = 0
SCOUT_ERR_INVALID_ARGUMENT = 1
SCOUT_ERR_LOGIC = 2
SCOUT_ERR_CUDA = 3
SCOUT_ERR_UNSUPPORTED = 4

SCOUT_F32, SCOUT_BF16, SCOUT_F64 = 0, 1, 2
SCOUT_GPU_SIDE_PREDICTED, SCOUT_GPU_SIDE_ALL_RESIDENT = 0, 1
SCOUT_DIGEST_MINMAX, SCOUT_DIGEST_MEAN = 0, 1
HEAD_DIM = 128
BLOCK_SIZE = 64

# every extern "C" symbol of include/scout_b200.h
EXPORTED = (
    "scout_last_error", "scout_version", "scout_slot_bytes",
    "scout_kv_write_tokens", "scout_kv_read_tokens", "scout_digest_build", "scout_kv_append",
    "scout_score_topk_split", "scout_score_topk_split_batch", "scout_sparse_decode_workspace_bytes",
    "scout_sparse_decode_grid",
    "scout_sparse_decode", "scout_merge_partials", "scout_recall_gather", "scout_recall_copy",
    "scout_engine_create", "scout_engine_destroy", "scout_engine_decode_step", "scout_engine_decode_step_host",
    "scout_engine_sync", "scout_engine_set_timing", "scout_engine_stats", "scout_engine_k2_times", "scout_engine_k1_outputs",
    "scout_tier_append", "scout_tier_apply", "scout_tier_schedule_recall", "scout_tier_plan", "scout_tier_mark",
    "scout_tier_place", "scout_tier_prefill", "scout_qpred_workspace_bytes", "scout_qpred_pack_weights", "scout_predict_query",
    "scout_recall_gather_ids", "scout_kv_writeback", "scout_engine_decode_step_kv", "scout_engine_recall_stats", "scout_engine_cpu_tokens", "scout_calibrate_intervals", "scout_engine_prefill",
    "scout_engine_overlap_stats", "scout_engine_set_overlap",
    "scout_engine_decode_step_kv_host", "scout_cpu_partial_attention", "scout_cpu_partial_attention_ex", "scout_cpu_coattn_kernel", "scout_engine_tier_changed",
    "scout_engine_worker_stats", "scout_engine_check_state", "scout_engine_decode_layer", "scout_engine_decode_layer_x",
)

_vp = C.c_void_p
_i32p = C.c_void_p  # device pointers travel as void*


class TierLayer(C.Structure):
    _fields_ = [("table", _vp), ("tier", _vp), ("last_sel", _vp), ("ready", _vp), ("ticket", _vp),
                ("free_slots", _vp), ("n_free", _vp), ("err", _vp), ("capacity", C.c_int),
                ("slots_per_unit", C.c_int), ("free_head", _vp), ("free_owner", _vp), ("warm", _vp)]


class TopkArgs(C.Structure):
    _fields_ = [
        ("n_units", C.c_int), ("group", C.c_int), ("digest_dtype", C.c_int), ("method", C.c_int),
        ("k", C.c_int), ("k_stride", C.c_int), ("nb_stride", C.c_int), ("step", C.c_int),
        ("q", _vp), ("digests", _vp), ("n_tokens", _vp), ("block_table", _vp),
        ("sel_ids", _vp), ("n_sel", _vp), ("res_slots", _vp), ("res_ids", _vp), ("n_res", _vp),
        ("cpu_ids", _vp), ("n_cpu", _vp), ("res_tokens", _vp), ("cpu_tokens", _vp),
        ("last_selected", _vp), ("scores_out", _vp), ("flags", C.c_int),
        ("done_flag", _vp), ("done_ctr", _vp), ("done_token", C.c_uint), ("q_dtype", C.c_int),
    ]


class DecodeArgs(C.Structure):
    _fields_ = [
        ("n_units", C.c_int), ("group", C.c_int), ("kv_dtype", C.c_int), ("k_stride", C.c_int),
        ("scale", C.c_float),
        ("q", _vp), ("kv_pool", _vp), ("res_slots", _vp), ("res_ids", _vp), ("n_res", _vp),
        ("n_tokens", _vp), ("cpu_o", _vp), ("cpu_ml", _vp), ("o", _vp), ("ml", _vp),
        ("workspace", _vp), ("workspace_bytes", C.c_size_t), ("max_ctas", C.c_int), ("flags", C.c_int),
        ("q_dtype", C.c_int),
    ]


class LayerDesc(C.Structure):
    _fields_ = [("digests", _vp), ("block_table", _vp), ("recall_src", _vp), ("recall_dst", _vp),
                ("recall_n", C.c_int)]


class EngineConfig(C.Structure):
    _fields_ = [
        ("layers", C.c_int), ("batch", C.c_int), ("hq", C.c_int), ("hkv", C.c_int), ("k", C.c_int),
        ("nb_stride", C.c_int), ("kv_dtype", C.c_int), ("scale", C.c_float), ("recall_interval", C.c_int),
        ("kv_pool", _vp), ("n_tokens", _vp), ("host_tier", _vp), ("max_ctas", C.c_int),
        ("host_staging", C.c_int), ("chunk_layers", C.c_int), ("recall_mode", C.c_int),
        ("q_dtype", C.c_int),
        ("tier", _vp), ("host_blocks", C.c_longlong), ("cpu_dtype", C.c_int),
        ("recall_intervals", _vp), ("recall_stagger", C.c_int), ("cpu_worker", C.c_int), ("cpu_threads", C.c_int),
        ("gpu_side_policy", C.c_int), ("layer_ctas", C.c_int), ("host_units", C.c_int), ("host_unit0", C.c_int),
        ("hidden", C.c_int),
    ]


class ScoutError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[scout status {code}] {msg}")
        self.code = code


_lib = None


def lib() -> C.CDLL:
    """Load libscout_b200.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(str(LIB_PATH))
        L.scout_last_error.restype = C.c_char_p
        L.scout_version.restype = C.c_int
        L.scout_slot_bytes.restype = C.c_size_t
        L.scout_slot_bytes.argtypes = [C.c_int]
        L.scout_kv_write_tokens.argtypes = [_vp, C.c_int, _vp, _vp, _vp, _vp, C.c_int, _vp]
        L.scout_kv_read_tokens.argtypes = [_vp, C.c_int, _vp, _vp, _vp, _vp, C.c_int, _vp]
        L.scout_digest_build.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, C.c_int, _vp]
        _tl = C.POINTER(TierLayer)
        L.scout_tier_append.argtypes = [_tl, C.c_int, C.c_int, _vp, C.c_int, _vp, _vp, _vp]
        L.scout_tier_apply.argtypes = [_tl, C.c_int, C.c_int, _vp, C.c_int, _vp, _vp]
        L.scout_tier_schedule_recall.argtypes = [_tl, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int, C.c_int, C.c_int,
                                                 _vp, _vp]
        L.scout_tier_plan.argtypes = [_tl, C.c_int, C.c_int, _vp, C.c_int, _vp, _vp]
        L.scout_tier_mark.argtypes = [_tl, C.c_int, C.c_int, _vp, _vp, C.c_int, C.c_int, _vp]
        L.scout_tier_place.argtypes = [_tl, C.c_int, C.c_int, _vp, _vp, _vp, C.c_int, _vp, _vp]
        L.scout_tier_prefill.argtypes = [_tl, C.c_int, C.c_int, _vp, C.c_int, _vp, _vp, C.c_int, _vp, C.c_int, _vp,
                                         _vp, C.c_longlong, C.c_longlong, _vp, _vp]
        L.scout_qpred_workspace_bytes.argtypes = [C.c_int] * 4
        L.scout_qpred_workspace_bytes.restype = C.c_size_t
        L.scout_qpred_pack_weights.argtypes = [_vp, C.c_int, C.c_int, _vp, _vp]
        L.scout_predict_query.argtypes = [_vp, C.c_int, C.c_int, _vp, C.c_int, _vp, _vp, _vp, C.c_size_t, C.c_int,
                                          _vp]
        L.scout_recall_gather_ids.argtypes = [_vp, C.c_int, _vp, C.c_longlong, C.c_int, C.c_longlong, C.c_int, _vp,
                                              _vp, _vp, C.c_int, C.c_int, _vp]
        L.scout_kv_writeback.argtypes = [_vp, C.c_int, _vp, C.c_longlong, C.c_int, C.c_longlong, C.c_int, _vp, _vp,
                                         _vp]
        L.scout_cpu_partial_attention.argtypes = [_vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp, C.c_int, C.c_float,
                                                  C.c_int, _vp, _vp, C.c_int]
        L.scout_cpu_partial_attention_ex.argtypes = [_vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp, C.c_int, C.c_int,
                                                     C.c_float, C.c_int, _vp, C.c_int, _vp, C.c_int]
        L.scout_cpu_coattn_kernel.argtypes = [C.c_int]
        L.scout_kv_append.argtypes = [_vp, C.c_int, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, C.c_int, C.c_int, _vp]
        L.scout_score_topk_split.argtypes = [C.POINTER(TopkArgs), _vp]
        L.scout_score_topk_split_batch.argtypes = [C.POINTER(TopkArgs), C.c_int, _vp]
        L.scout_sparse_decode_workspace_bytes.restype = C.c_size_t
        L.scout_sparse_decode_workspace_bytes.argtypes = [C.c_int, C.c_int, C.c_int]
        L.scout_sparse_decode_grid.argtypes = [C.c_int, C.c_int, C.c_int]
        L.scout_sparse_decode.argtypes = [C.POINTER(DecodeArgs), _vp]
        L.scout_merge_partials.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, C.c_int, _vp]
        L.scout_recall_gather.argtypes = [_vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp]
        L.scout_recall_copy.argtypes = [_vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp]
        L.scout_engine_create.argtypes = [C.POINTER(EngineConfig), C.POINTER(LayerDesc), C.POINTER(_vp)]
        L.scout_engine_destroy.argtypes = [_vp]
        L.scout_engine_decode_step.argtypes = [_vp, C.c_int] + [_vp] * 6 + [_vp]
        L.scout_engine_decode_step_kv.argtypes = [_vp, C.c_int] + [_vp] * 8 + [_vp]
        L.scout_engine_decode_step_kv_host.argtypes = [_vp, C.c_int] + [_vp] * 10 + [_vp]
        L.scout_engine_decode_step_host.argtypes = [_vp, C.c_int] + [_vp] * 8 + [_vp]
        L.scout_engine_sync.argtypes = [_vp, _vp]
        L.scout_engine_tier_changed.argtypes = [_vp]
        L.scout_engine_set_timing.argtypes = [_vp, C.c_int]
        L.scout_engine_stats.argtypes = [_vp, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_longlong)]
        L.scout_engine_k2_times.argtypes = [_vp, _vp, C.c_int, C.POINTER(C.c_int)]
        L.scout_engine_recall_stats.argtypes = [_vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong), C.c_int]
        L.scout_engine_cpu_tokens.argtypes = [_vp, _vp, _vp]
        L.scout_engine_prefill.argtypes = [_vp, _vp, _vp, _vp, C.c_int, _vp, _vp]
        L.scout_engine_overlap_stats.argtypes = [_vp, _vp, _vp, C.c_int]
        L.scout_engine_set_overlap.argtypes = [_vp, C.c_int]
        L.scout_calibrate_intervals.argtypes = [_vp, _vp, C.c_int, C.c_int, C.c_double, _vp]
        L.scout_engine_k1_outputs.argtypes = [_vp] + [C.POINTER(_vp)] * 7
        L.scout_engine_worker_stats.argtypes = [_vp, C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.scout_engine_check_state.argtypes = [_vp]
        L.scout_engine_decode_layer.argtypes = [_vp, C.c_int, C.c_int] + [_vp] * 8 + [_vp]
        L.scout_engine_decode_layer_x.argtypes = [_vp, C.c_int, C.c_int] + [_vp] * 9 + [_vp]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != SCOUT_OK:
        msg = lib().scout_last_error().decode()
        if rc == SCOUT_ERR_INVALID_ARGUMENT:
            raise ValueError(msg)  # std::invalid_argument in the reference
        raise ScoutError(rc, msg)
