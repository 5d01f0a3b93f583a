"""Python handle on the C++ decode-step engine (csrc/engine.cpp, C ABI
scout_engine_*): the GPU side of ScoutEngine::decode_step
(reference proj/include/scout/engine.hpp:205-314).

The engine is C++; this class only passes device / pinned-host pointers and
the current torch stream. Tier policy (tables, recall plans) is owned by the
caller, as in the reference where it lives in TieredKvCache / recall.hpp.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _capi as A
from . import ops


@dataclass
class LayerState:
    digests: torch.Tensor                     # [U][2][128][nbs] kv dtype
    table: torch.Tensor                       # [U][nbs] int32 slot or -1 (planning view)
    recall_src: torch.Tensor | None = None    # [n] int64 host block index (CPU tensor)
    recall_dst: torch.Tensor | None = None    # [n] int32 pool slot (CPU tensor)


def _p(t):
    return None if t is None else t.data_ptr()


class DecodeEngine:
    def __init__(self, *, layers, batch, hq, hkv, k, n_tokens, pool, kv_dtype, layer_states, scale,
                 recall_interval=0, host_tier=None, max_ctas=0, host_staging=False, chunk_layers=8,
                 recall_mode=1, q_dtype=torch.float32, tier=None, host_blocks=0, cpu_dtype=torch.float32,
                 recall_intervals=None, recall_stagger=False, cpu_worker=False, cpu_threads=0,
                 gpu_side_policy="predicted_topk_intersect_resident", layer_ctas=0, host_units=0, host_unit0=0,
                 hidden=0):
        """tier: a tier.DeviceTieredCache whose state the engine drives on the
        device (device tier mode: decode_step_kv); host_tier then holds block
        images at ((layer*U + unit)*nb_stride + id) % host_blocks.
        recall_intervals: per-layer recall intervals (engine.hpp:35; default:
        recall_interval for every layer), triggered as the reference does
        (step - last_recall >= interval, recall.hpp:114-126); recall_stagger:
        round 1's (step + layer) % interval cadence instead.
        cpu_worker: the engine computes each step's CPU partials itself
        (device tier mode, host path; the decode calls then take no cpu_o /
        cpu_ml) on cpu_threads host threads (0 = all).
        gpu_side_policy: the reference's GpuSidePolicy (engine.hpp:25-29):
        "predicted_topk_intersect_resident" or "all_resident" (the GPU side
        attends to the layer's whole fast tier at attention time).
        layer_ctas: K2 CTAs of a layer-by-layer launch (0 automatic, < 0 all).
        hidden: the model's hidden size for decode_layer_x (the layer-ahead
        q prediction, K6, inside the layer-by-layer mode); 0 = off.
        host_units / host_unit0: the host tier's unit index space when ranks
        share one (image ((layer*host_units + host_unit0 + u)*nb_stride + id)
        % host_blocks); 0 / 0: this engine's units."""
        self.L, self.batch, self.hq, self.hkv, self.G, self.k = layers, batch, hq, hkv, hq // hkv, k
        self.U = batch * hkv
        self.layer_states = layer_states  # keep tensors alive
        self.n_tokens = n_tokens
        self.pool, self.host_tier = pool, host_tier
        cfg = A.EngineConfig()
        cfg.layers, cfg.batch, cfg.hq, cfg.hkv, cfg.k = layers, batch, hq, hkv, k
        cfg.nb_stride = int(layer_states[0].digests.shape[-1])
        cfg.kv_dtype = ops.dtype_code(kv_dtype)
        cfg.scale = float(scale)
        cfg.recall_interval = int(recall_interval)
        cfg.kv_pool, cfg.n_tokens, cfg.host_tier = _p(pool), _p(n_tokens), _p(host_tier)
        cfg.max_ctas, cfg.host_staging, cfg.chunk_layers = int(max_ctas), int(host_staging), int(chunk_layers)
        cfg.recall_mode = int(recall_mode)
        cfg.q_dtype = ops.dtype_code(q_dtype)
        cfg.cpu_dtype = ops.dtype_code(cpu_dtype)  # CPU-partial o: f32 or bf16
        if recall_intervals is not None:
            self._rc_int = (C.c_int32 * layers)(*[int(x) for x in recall_intervals])
            cfg.recall_intervals = C.cast(self._rc_int, C.c_void_p)
        cfg.recall_stagger = int(bool(recall_stagger))
        cfg.cpu_worker, cfg.cpu_threads = int(bool(cpu_worker)), int(cpu_threads)
        policies = {"predicted_topk_intersect_resident": A.SCOUT_GPU_SIDE_PREDICTED,
                    "all_resident": A.SCOUT_GPU_SIDE_ALL_RESIDENT}
        if gpu_side_policy not in policies:
            raise ValueError(f"gpu_side_policy {gpu_side_policy!r}: one of {sorted(policies)}")
        cfg.gpu_side_policy = policies[gpu_side_policy]
        cfg.layer_ctas = int(layer_ctas)
        cfg.host_units, cfg.host_unit0 = int(host_units), int(host_unit0)
        cfg.hidden = int(hidden)
        self.gpu_side_policy = gpu_side_policy
        self.cpu_worker = bool(cpu_worker)
        self.tier = tier
        if tier is not None:
            self._tier_descs = (A.TierLayer * layers)(*[tier.layer_desc(i) for i in range(layers)])
            cfg.tier = C.cast(self._tier_descs, C.c_void_p)
            cfg.host_blocks = int(host_blocks)
        self.q_dtype = q_dtype
        self.cpu_dtype = cpu_dtype
        descs = (A.LayerDesc * layers)()
        for i, st in enumerate(layer_states):
            descs[i].digests, descs[i].block_table = _p(st.digests), _p(st.table)
            if st.recall_src is not None:
                assert st.recall_src.device.type == "cpu" and st.recall_dst.device.type == "cpu"
                descs[i].recall_src, descs[i].recall_dst = _p(st.recall_src), _p(st.recall_dst)
                descs[i].recall_n = int(st.recall_dst.numel())
        h = C.c_void_p()
        A.check(A.lib().scout_engine_create(C.byref(cfg), descs, C.byref(h)))
        self._h = h

    def close(self):
        """Destroy the engine (drains its recall thread); idempotent."""
        h = getattr(self, "_h", None)
        if h:
            self._h = None
            A.lib().scout_engine_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the module globals may be gone already
            pass

    @staticmethod
    def _stream():
        return torch.cuda.current_stream().cuda_stream

    def _check(self, q_true, q_pred, cpu_o, cpu_ml):
        """The buffers' element types must be the engine's (the C ABI takes raw
        pointers: a bf16 tensor read as f32 would be garbage, not an error)."""
        for name, t, dt in (("q_true", q_true, self.q_dtype), ("q_pred", q_pred, self.q_dtype),
                            ("cpu_o", cpu_o, self.cpu_dtype), ("cpu_ml", cpu_ml, torch.float32)):
            if t is not None and t.dtype != dt:
                raise ValueError(f"{name}: dtype {t.dtype}, the engine was configured for {dt}")
        if self.cpu_worker and (cpu_o is not None or cpu_ml is not None):
            raise ValueError("cpu_worker engine: the CPU partials are computed inside, pass cpu_o = cpu_ml = None")

    def decode_step(self, step, q_true, q_pred, cpu_o, cpu_ml, out_o, out_ml):
        """Device tensors: q_true/q_pred [L][U*G][128] (q dtype), cpu_o [L][U*G][128] (cpu dtype),
        out_o [L][U*G][128] f32, cpu_ml/out_ml [L][U*G][2] f32."""
        self._check(q_true, q_pred, cpu_o, cpu_ml)
        A.check(A.lib().scout_engine_decode_step(self._h, int(step), _p(q_true), _p(q_pred), _p(cpu_o), _p(cpu_ml),
                                                 _p(out_o), _p(out_ml), self._stream()))

    def decode_step_kv(self, step, q_true, q_pred, cpu_o, cpu_ml, k_new, v_new, out_o, out_ml):
        """Device tier mode: the step appends k_new / v_new [L][U][128] f32."""
        self._check(q_true, q_pred, cpu_o, cpu_ml)
        A.check(A.lib().scout_engine_decode_step_kv(self._h, int(step), _p(q_true), _p(q_pred), _p(cpu_o), _p(cpu_ml),
                                                    _p(k_new), _p(v_new), _p(out_o), _p(out_ml), self._stream()))

    def decode_step_kv_host(self, step, h_q_true, h_q_pred, h_cpu_o, h_cpu_ml, h_k_new, h_v_new, h_out_o, h_out_ml,
                            h_cpu_ids=None, h_n_cpu=None):
        """Device tier mode from pinned host tensors (+ the token's K/V rows)."""
        self._check(h_q_true, h_q_pred, h_cpu_o, h_cpu_ml)
        A.check(A.lib().scout_engine_decode_step_kv_host(self._h, int(step), _p(h_q_true), _p(h_q_pred), _p(h_cpu_o),
                                                         _p(h_cpu_ml), _p(h_k_new), _p(h_v_new), _p(h_out_o),
                                                         _p(h_out_ml), _p(h_cpu_ids), _p(h_n_cpu), self._stream()))

    def decode_step_host(self, step, h_q_true, h_q_pred, h_cpu_o, h_cpu_ml, h_out_o, h_out_ml, h_cpu_ids=None,
                         h_n_cpu=None):
        """Pinned host tensors, same layouts; h_cpu_ids [L][U][k], h_n_cpu [L][U] int32."""
        self._check(h_q_true, h_q_pred, h_cpu_o, h_cpu_ml)
        A.check(A.lib().scout_engine_decode_step_host(self._h, int(step), _p(h_q_true), _p(h_q_pred), _p(h_cpu_o),
                                                      _p(h_cpu_ml), _p(h_out_o), _p(h_out_ml), _p(h_cpu_ids),
                                                      _p(h_n_cpu), self._stream()))

    def decode_layer(self, step, layer, q_true, q_pred_next, cpu_o, cpu_ml, k_new, v_new, out_o, out_ml):
        """Layer-by-layer device tier mode: one layer of a step (layers 0..L-1 in
        order); q_true [U*G][128] of this layer, q_pred_next of the next (None
        for the last layer), k_new / v_new [U][128] f32; outputs [U*G][128] / [U*G][2]."""
        self._check(q_true, q_pred_next, cpu_o, cpu_ml)
        A.check(A.lib().scout_engine_decode_layer(self._h, int(step), int(layer), _p(q_true), _p(q_pred_next),
                                                  _p(cpu_o), _p(cpu_ml), _p(k_new), _p(v_new), _p(out_o), _p(out_ml),
                                                  self._stream()))

    def decode_layer_x(self, step, layer, q_true, x_next, wq_next, cpu_o, cpu_ml, k_new, v_new, out_o, out_ml):
        """decode_layer with the next layer's q_pred predicted inside the engine
        (engine.hpp:237): x_next [batch][hidden] f32 and wq_next, an
        ops.QueryPredictor's packed W_Q of layer + 1 (its w_packed), or None
        for the last layer."""
        self._check(q_true, None, cpu_o, cpu_ml)
        wp = None if wq_next is None else (wq_next.w_packed if hasattr(wq_next, "w_packed") else wq_next)
        A.check(A.lib().scout_engine_decode_layer_x(self._h, int(step), int(layer), _p(q_true), _p(x_next), _p(wp),
                                                    _p(cpu_o), _p(cpu_ml), _p(k_new), _p(v_new), _p(out_o),
                                                    _p(out_ml), self._stream()))

    def tier_changed(self):
        """The tier state was changed outside the engine: plan the next step afresh."""
        A.check(A.lib().scout_engine_tier_changed(self._h))

    def sync(self):
        A.check(A.lib().scout_engine_sync(self._h, self._stream()))

    def set_timing(self, on: bool):
        A.check(A.lib().scout_engine_set_timing(self._h, int(on)))

    def recall_stats(self, reset=False):
        """Device tier mode: (recalled blocks served by a warm image in HBM,
        recalled blocks copied from the host tier) since the last reset."""
        w, c = C.c_longlong(0), C.c_longlong(0)
        A.check(A.lib().scout_engine_recall_stats(self._h, C.byref(w), C.byref(c), int(bool(reset))))
        return int(w.value), int(c.value)

    def prefill(self, k_rows, v_rows, n_tokens, q_place=None):
        """ScoutEngine::prefill + place_after_prefill (engine.hpp:192-201) on
        fresh tier state: k_rows / v_rows [L][U][T][128] f32 device, n_tokens
        [U], q_place [L][U*G][128] (q dtype) or None."""
        k = k_rows.float().contiguous()
        v = v_rows.float().contiguous()
        nt = n_tokens.to(device=k.device, dtype=torch.int32).contiguous()
        qp = None if q_place is None else q_place.contiguous()
        A.check(A.lib().scout_engine_prefill(self._h, _p(k), _p(v), _p(nt), int(k.shape[2]), _p(qp), self._stream()))

    def set_overlap(self, k1_sms: int):
        """The overlapped step's K1 share: -1 environment / default, 0 off, > 0 SMs."""
        A.check(A.lib().scout_engine_set_overlap(self._h, int(k1_sms)))

    def overlap_stats(self, reset=False):
        """(steps run with K1 beside K2 since the last reset, K1's SM share of
        the last one): scout_engine_overlap_stats."""
        n, sms = C.c_longlong(0), C.c_int(0)
        A.check(A.lib().scout_engine_overlap_stats(self._h, C.byref(n), C.byref(sms), int(bool(reset))))
        return int(n.value), int(sms.value)

    def cpu_tokens(self):
        """(cpu tokens per layer summed over the units, budget U * k * 64) of the
        last step: one RatioTrace sample per layer (engine.hpp:283)."""
        cpu = (C.c_int64 * self.L)()
        bud = (C.c_int64 * self.L)()
        A.check(A.lib().scout_engine_cpu_tokens(self._h, C.cast(cpu, C.c_void_p), C.cast(bud, C.c_void_p)))
        return list(cpu), list(bud)

    def k2_times(self, max_n=4096):
        """Per-launch K2 durations (ms) of the current timing window (before stats())."""
        buf = (C.c_float * max_n)()
        n = C.c_int()
        A.check(A.lib().scout_engine_k2_times(self._h, C.cast(buf, C.c_void_p), max_n, C.byref(n)))
        return list(buf[:min(n.value, max_n)])

    def stats(self):
        ms, n, launches = C.c_double(), C.c_int(), C.c_longlong()
        A.check(A.lib().scout_engine_stats(self._h, C.byref(ms), C.byref(n), C.byref(launches)))
        return ms.value, n.value, launches.value

    def check_state(self):
        """Raise on the tier state's sticky errors (rejected recall ticket, out of
        slots, check_split violated); synchronises."""
        A.check(A.lib().scout_engine_check_state(self._h))

    def worker_stats(self):
        """In-engine CPU worker: (CPU ms summed over the steps since the last call, steps)."""
        ms, n = C.c_double(), C.c_int()
        A.check(A.lib().scout_engine_worker_stats(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def k1_outputs(self):
        """Zero-copy torch views of the engine's per-layer K1 outputs (device)."""
        ptrs = [C.c_void_p() for _ in range(7)]
        A.check(A.lib().scout_engine_k1_outputs(self._h, *[C.byref(p) for p in ptrs]))
        L, U, k = self.L, self.U, self.k
        names = ["res_slots", "res_ids", "n_res", "cpu_ids", "n_cpu", "res_tokens", "cpu_tokens"]
        shapes = [(L, U, k), (L, U, k), (L, U), (L, U, k), (L, U), (L, U), (L, U)]
        return {n: torch.as_tensor(_DeviceArray(p.value, sh), device=self.pool.device)
                for n, p, sh in zip(names, ptrs, shapes)}


class _DeviceArray:
    """__cuda_array_interface__ over engine-owned int32 device memory."""

    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<i4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


__all__ = ["DecodeEngine", "LayerState"]


def calibrate_intervals(cpu_tokens, budget_tokens, beta=0.12):
    """calibrate_intervals (recall.hpp:66-95) on a recall-free trace:
    cpu_tokens / budget_tokens [layers][steps] -> per-layer intervals."""
    import numpy as np

    cpu = np.ascontiguousarray(cpu_tokens, dtype=np.int64)
    bud = np.ascontiguousarray(budget_tokens, dtype=np.int64)
    L, S = cpu.shape
    out = np.zeros(L, dtype=np.int32)
    A.check(A.lib().scout_calibrate_intervals(cpu.ctypes.data, bud.ctypes.data, L, S, float(beta), out.ctypes.data))
    return out.tolist()
