"""Torch-tensor entry points over the C ABI (device memory / streams only).

Each function launches on torch's current CUDA stream and returns device
tensors; torch is plumbing here, every computation is one of the sm_100a
kernels in csrc/. Layouts are those of include/scout_b200.h.
"""
from __future__ import annotations

import math

import torch

from . import _capi as A

_DTYPE_CODE = {torch.float32: A.SCOUT_F32, torch.bfloat16: A.SCOUT_BF16, torch.float64: A.SCOUT_F64}


def _p(t):
    return None if t is None else t.data_ptr()


def _stream():
    return torch.cuda.current_stream().cuda_stream


def dtype_code(dt: torch.dtype) -> int:
    return _DTYPE_CODE[dt]


def slot_bytes(kv_dtype: torch.dtype) -> int:
    return int(A.lib().scout_slot_bytes(dtype_code(kv_dtype)))


def alloc_pool(n_slots: int, kv_dtype: torch.dtype, device="cuda") -> torch.Tensor:
    """KV pool: n_slots blocks of (K, V) 64 x 128 in the kernel layout (raw bytes)."""
    return torch.empty(n_slots * slot_bytes(kv_dtype), dtype=torch.uint8, device=device)


def _i32(x, device):
    return torch.as_tensor(x, dtype=torch.int32, device=device).contiguous()


def kv_write_tokens(pool, kv_dtype, slots, rows, k_rows, v_rows):
    dev = pool.device
    slots, rows = _i32(slots, dev), _i32(rows, dev)
    k_rows = k_rows.to(device=dev, dtype=torch.float32).contiguous()
    v_rows = v_rows.to(device=dev, dtype=torch.float32).contiguous()
    A.check(A.lib().scout_kv_write_tokens(_p(pool), dtype_code(kv_dtype), _p(slots), _p(rows), _p(k_rows),
                                          _p(v_rows), int(slots.numel()), _stream()))


def kv_read_tokens(pool, kv_dtype, slots, rows):
    dev = pool.device
    slots, rows = _i32(slots, dev), _i32(rows, dev)
    n = int(slots.numel())
    k = torch.empty(n, A.HEAD_DIM, dtype=torch.float32, device=dev)
    v = torch.empty_like(k)
    A.check(A.lib().scout_kv_read_tokens(_p(pool), dtype_code(kv_dtype), _p(slots), _p(rows), _p(k), _p(v), n,
                                         _stream()))
    return k, v


def write_blocks(pool, kv_dtype, slots, keys, values):
    """Write whole blocks: keys/values [n][rows<=64][128] -> slots[n] (rows 0..)."""
    n, rows = keys.shape[0], keys.shape[1]
    dev = pool.device
    sl = _i32(slots, dev).repeat_interleave(rows)
    rr = torch.arange(rows, device=dev, dtype=torch.int32).repeat(n)
    kv_write_tokens(pool, kv_dtype, sl, rr, keys.reshape(-1, A.HEAD_DIM), values.reshape(-1, A.HEAD_DIM))


def digest_build(pool, kv_dtype, method, slots, block_rows, units, block_ids, digests, nb_stride):
    dev = pool.device
    slots, block_rows, units, block_ids = (_i32(x, dev) for x in (slots, block_rows, units, block_ids))
    A.check(A.lib().scout_digest_build(_p(pool), dtype_code(kv_dtype), int(method), int(slots.numel()), _p(slots),
                                       _p(block_rows), _p(units), _p(block_ids), _p(digests), int(nb_stride),
                                       _stream()))


def kv_append(pool, kv_dtype, method, open_slot, n_tokens, k_rows, v_rows, digests, nb_stride, advance=True):
    """append_token (kv_store.hpp:90-117) for one layer of every unit: rows to
    the open block, digest column updated in place, n_tokens advanced."""
    dev = pool.device
    open_slot = _i32(open_slot, dev)
    assert n_tokens.dtype == torch.int32 and n_tokens.device == dev
    k_rows = torch.as_tensor(k_rows, dtype=torch.float32, device=dev).contiguous()
    v_rows = torch.as_tensor(v_rows, dtype=torch.float32, device=dev).contiguous()
    A.check(A.lib().scout_kv_append(_p(pool), dtype_code(kv_dtype), int(method), int(open_slot.numel()),
                                    _p(open_slot), _p(n_tokens), _p(k_rows), _p(v_rows), _p(digests),
                                    int(nb_stride), int(bool(advance)), _stream()))


def score_topk_split(q, digests, n_tokens, k, group, *, method=A.SCOUT_DIGEST_MINMAX, block_table=None, step=0,
                     k_stride=None, want_scores=False, last_selected=None, out=None):
    """K1. q [units*G][128] (f32 or bf16, or f64 for f64 digests); digests [units][2|1][128][nb_stride].

    Returns a dict of device tensors: sel_ids/n_sel, and when block_table is given
    res_slots/res_ids/n_res, cpu_ids/n_cpu, res_tokens/cpu_tokens (+ scores)."""
    dev = digests.device
    n_units = int(n_tokens.numel())
    nb_stride = int(digests.shape[-1])
    ks = int(k_stride or max(int(k), 1))
    o = out if out is not None else {}

    def buf(name, shape, dt=torch.int32):
        if name not in o:
            o[name] = torch.empty(shape, dtype=dt, device=dev)
        return o[name]

    args = A.TopkArgs()
    args.n_units, args.group, args.digest_dtype, args.method = n_units, int(group), dtype_code(digests.dtype), int(method)
    args.k, args.k_stride, args.nb_stride, args.step = int(k), ks, nb_stride, int(step)
    args.q, args.digests, args.n_tokens = _p(q), _p(digests), _p(n_tokens)
    args.q_dtype = A.SCOUT_BF16 if q.dtype == torch.bfloat16 else A.SCOUT_F32
    args.sel_ids, args.n_sel = _p(buf("sel_ids", (n_units, ks))), _p(buf("n_sel", (n_units,)))
    if block_table is not None:
        args.block_table = _p(block_table)
        args.res_slots, args.res_ids = _p(buf("res_slots", (n_units, ks))), _p(buf("res_ids", (n_units, ks)))
        args.n_res, args.cpu_ids = _p(buf("n_res", (n_units,))), _p(buf("cpu_ids", (n_units, ks)))
        args.n_cpu = _p(buf("n_cpu", (n_units,)))
        args.res_tokens, args.cpu_tokens = _p(buf("res_tokens", (n_units,))), _p(buf("cpu_tokens", (n_units,)))
    if last_selected is not None:
        args.last_selected = _p(last_selected)
    if want_scores:
        args.scores_out = _p(buf("scores", (n_units, nb_stride), torch.float64))
    A.check(A.lib().scout_score_topk_split(args, _stream()))
    return o


class DecodeWorkspace:
    """Caller-owned K2 workspace (zeroed once; kernels leave counters zeroed)."""

    def __init__(self, n_units: int, group: int, device="cuda", max_ctas: int = 0):
        nbytes = int(A.lib().scout_sparse_decode_workspace_bytes(n_units, group, max_ctas))
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        self.n_units, self.max_ctas = n_units, max_ctas


def sparse_decode(q, pool, kv_dtype, res_slots, res_ids, n_res, n_tokens, group, scale=None, *, cpu_o=None,
                  cpu_ml=None, o=None, ml=None, workspace=None, max_ctas=0):
    """K2 (+K3 fused). Returns (o [units*G][128] f32, ml [units*G][2] f32)."""
    dev = q.device
    n_units = int(n_tokens.numel())
    if scale is None:
        scale = 1.0 / math.sqrt(A.HEAD_DIM)
    if o is None:
        o = torch.empty(n_units * group, A.HEAD_DIM, dtype=torch.float32, device=dev)
    if ml is None:
        ml = torch.empty(n_units * group, 2, dtype=torch.float32, device=dev)
    if workspace is None or workspace.n_units < n_units or workspace.max_ctas != max_ctas:
        workspace = DecodeWorkspace(n_units, group, dev, max_ctas)
    args = A.DecodeArgs()
    args.n_units, args.group, args.kv_dtype, args.k_stride = n_units, int(group), dtype_code(kv_dtype), int(res_slots.shape[-1])
    args.scale = float(scale)
    args.q, args.kv_pool, args.res_slots, args.res_ids = _p(q), _p(pool), _p(res_slots), _p(res_ids)
    args.q_dtype = A.SCOUT_BF16 if q.dtype == torch.bfloat16 else A.SCOUT_F32
    args.n_res, args.n_tokens, args.cpu_o, args.cpu_ml = _p(n_res), _p(n_tokens), _p(cpu_o), _p(cpu_ml)
    args.o, args.ml = _p(o), _p(ml)
    args.workspace, args.workspace_bytes, args.max_ctas = _p(workspace.buf), workspace.buf.numel(), int(max_ctas)
    A.check(A.lib().scout_sparse_decode(args, _stream()))
    return o, ml


def cpu_coattn_kernel(kv_dtype=torch.bfloat16):
    """The CPU worker's kernel for kv_dtype here: "amx-bf16", "avx512-f32" or "scalar"."""
    return {2: "amx-bf16", 1: "avx512-f32", 0: "scalar"}[A.lib().scout_cpu_coattn_kernel(dtype_code(kv_dtype))]


def merge_partials(a_o, a_ml, b_o, b_ml, out_o=None, out_ml=None):
    n = int(a_o.shape[0])
    out_o = torch.empty_like(a_o) if out_o is None else out_o
    out_ml = torch.empty_like(a_ml) if out_ml is None else out_ml
    A.check(A.lib().scout_merge_partials(_p(a_o), _p(a_ml), _p(b_o), _p(b_ml), _p(out_o), _p(out_ml), n, _stream()))
    return out_o, out_ml


def recall_gather(pool, kv_dtype, host_blocks, src_index, dst_slots):
    """K4. host_blocks: pinned CPU uint8 tensor of block images (slot layout)."""
    dev = pool.device
    src = torch.as_tensor(src_index, dtype=torch.int64, device=dev).contiguous()
    dst = _i32(dst_slots, dev)
    A.check(A.lib().scout_recall_gather(_p(pool), dtype_code(kv_dtype), _p(host_blocks), _p(src), _p(dst),
                                        int(dst.numel()), _stream()))


def recall_copy(pool, kv_dtype, host_blocks, src_index, dst_slots):
    """K4 on the copy engines. src_index / dst_slots: host (CPU) arrays."""
    src = torch.as_tensor(src_index, dtype=torch.int64).contiguous()
    dst = torch.as_tensor(dst_slots, dtype=torch.int32).contiguous()
    A.check(A.lib().scout_recall_copy(_p(pool), dtype_code(kv_dtype), _p(host_blocks), _p(src), _p(dst),
                                      int(dst.numel()), _stream()))


class QueryPredictor:
    """K6: q_pred = predict_next_query(rms_normalize(x), W) (model.hpp:215-217)
    on the tcgen05 tensor cores. W [hidden][n_out] (the reference's layout) is
    packed once at construction."""

    def __init__(self, w: torch.Tensor, batch: int, max_ctas: int = 0):
        self.hidden, self.n_out = int(w.shape[0]), int(w.shape[1])
        self.dev = w.device
        w = w.to(torch.bfloat16).contiguous()
        self.w_packed = torch.empty_like(w)
        A.check(A.lib().scout_qpred_pack_weights(_p(w), self.hidden, self.n_out, _p(self.w_packed), _stream()))
        self.batch, self.max_ctas = batch, max_ctas
        nbytes = int(A.lib().scout_qpred_workspace_bytes(self.hidden, self.n_out, batch, max_ctas))
        self.ws = torch.zeros(nbytes, dtype=torch.uint8, device=self.dev)

    def __call__(self, x: torch.Tensor, out_f32=None, out_bf16=None, want=("f32",)):
        x = x.to(device=self.dev, dtype=torch.float32).contiguous()
        b = int(x.shape[0])
        assert b <= self.batch
        if out_f32 is None and "f32" in want:
            out_f32 = torch.empty(b, self.n_out, dtype=torch.float32, device=self.dev)
        if out_bf16 is None and "bf16" in want:
            out_bf16 = torch.empty(b, self.n_out, dtype=torch.bfloat16, device=self.dev)
        A.check(A.lib().scout_predict_query(_p(x), b, self.hidden, _p(self.w_packed), self.n_out, _p(out_f32),
                                            _p(out_bf16), _p(self.ws), self.ws.numel(), self.max_ctas, _stream()))
        return out_f32 if out_bf16 is None else (out_bf16 if out_f32 is None else (out_f32, out_bf16))


def cpu_partial_attention(host_tier, kv_dtype, host_index, n_blocks, q, group, scale=None, block_rows=None,
                          threads=0):
    """CPU co-attention worker (host tensors): unit u's heads over its blocks
    host_index[u, :n_blocks[u]] of the host tier. Returns (o, ml) host f32."""
    host_index = torch.as_tensor(host_index, dtype=torch.int64).contiguous()
    n_blocks = torch.as_tensor(n_blocks, dtype=torch.int32).contiguous()
    q = torch.as_tensor(q, dtype=torch.float32).contiguous()
    n_units = int(n_blocks.numel())
    if scale is None:
        scale = 1.0 / math.sqrt(A.HEAD_DIM)
    rows = None if block_rows is None else torch.as_tensor(block_rows, dtype=torch.int32).contiguous()
    o = torch.empty(n_units * group, A.HEAD_DIM, dtype=torch.float32)
    ml = torch.empty(n_units * group, 2, dtype=torch.float32)
    A.check(A.lib().scout_cpu_partial_attention(host_tier.data_ptr(), dtype_code(kv_dtype), host_index.data_ptr(),
                                                None if rows is None else rows.data_ptr(), n_blocks.data_ptr(),
                                                int(host_index.shape[1]), q.data_ptr(), int(group), float(scale),
                                                n_units, o.data_ptr(), ml.data_ptr(), int(threads)))
    return o, ml


def cpu_partial_attention_ex(host_tier, kv_dtype, host_index, n_blocks, q, group, o_dtype=torch.bfloat16, scale=None,
                             block_rows=None, threads=0):
    """scout_cpu_partial_attention_ex: as cpu_partial_attention with the query
    in its own dtype (f32 / bf16 host tensor) and o in o_dtype. Returns
    (o, ml) host tensors, o in o_dtype, ml f32."""
    host_index = torch.as_tensor(host_index, dtype=torch.int64).contiguous()
    n_blocks = torch.as_tensor(n_blocks, dtype=torch.int32).contiguous()
    q = q.contiguous()
    n_units = int(n_blocks.numel())
    if scale is None:
        scale = 1.0 / math.sqrt(A.HEAD_DIM)
    rows = None if block_rows is None else torch.as_tensor(block_rows, dtype=torch.int32).contiguous()
    o = torch.empty(n_units * group, A.HEAD_DIM, dtype=o_dtype)
    ml = torch.empty(n_units * group, 2, dtype=torch.float32)
    A.check(A.lib().scout_cpu_partial_attention_ex(host_tier.data_ptr(), dtype_code(kv_dtype), host_index.data_ptr(),
                                                   None if rows is None else rows.data_ptr(), n_blocks.data_ptr(),
                                                   int(host_index.shape[1]), q.data_ptr(), dtype_code(q.dtype),
                                                   int(group), float(scale), n_units, o.data_ptr(), dtype_code(o_dtype),
                                                   ml.data_ptr(), int(threads)))
    return o, ml
