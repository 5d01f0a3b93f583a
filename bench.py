#!/usr/bin/env python
"""Benchmark: ScoutAttention GPU-side sparse decode at Qwen3-32B shape, 32K context.

Default (--tier device): the complete decode step of ScoutEngine::decode_step
(engine.hpp:220-307) on the device: residency planning, select + mark,
begin_layer's ticket application, attention + LSE merge, append of the
token's K/V with digest refresh (seal write-through, LRU eviction), and the
periodic recall (the reference's cadence and set: maybe_schedule_recall,
recall.hpp:114-126). --tier static is the kernel view: residency fixed at the
paper's 8.2% CPU share, no appends.

Workload (BASELINE.json configs[2], the metric's config): 64 layers, 64 query /
8 KV heads, head_dim 128, batch 32 per GPU, 32K-token context (512 blocks of
64 tokens per (request, KV head)), top-64 block selection, bf16 KV, layer-ahead
CPU partials merged on the GPU, periodic recall every 16 steps. A "step" = one
decode token for every request: for each of the 64 layers, K1 (score + top-k +
split of layer i+1 with the predicted query) and K2+K3 (sparse flash-decode of
layer i over its resident selected blocks, fused LSE merge with the CPU
partial), plus the post-attention bookkeeping and the recall copies.

  value : decode tokens/s (all GPUs), inputs resident in HBM
  e2e   : same metric through the engine with HOST (pinned) inputs/outputs:
          per-step H2D of q_true, q_pred, CPU partials, new K/V; D2H of the
          attention output and the CPU-side block ids, inside the timed region
  e2e_with_cpu_worker : the composed step: the engine's own CPU worker
          computes every layer's CPU partial during the step from the ids K1
          just selected (no pre-staged partials)
  verify: one more step re-derived in float64 on the device for a sample of
          (layer, unit) pairs (top-k sets, split, attention)
  roofline: K2 (dominant kernel) algorithmic bytes / its CUDA-event time
  cpu_baseline: the reference's own C++ functions (oracle/_ref) on this host's
          cores over a bounded sample of the same workload

`--impl reference` times the reference CPU implementation alone (rank 0).
Multi-GPU: one process per GPU, requests sharded (weak scaling: 32 per GPU;
--global-batch: strong), every rank's shard a slice of one seeded global
workload; no collective on the path; timing = max over ranks; outside the
timed region rank 0 recomputes a sample of every rank's requests alone and
compares the outputs.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

D, BS = 128, 64
CONFIGS = {
    # BASELINE.json configs[2] (the metric's config) and configs[3] (sharded: --global-batch 128)
    "qwen3-32b-32k": dict(layers=64, hq=64, hkv=8, batch=32, ctx=32768, k=64, capacity=64, headroom=8,
                          recall=16, cpu_frac=0.082, hidden=5120),
    # configs[1]: Qwen3-8B, batch 16, 16K, GPU cache = 25% of the 256 blocks
    "qwen3-8b-16k": dict(layers=36, hq=32, hkv=8, batch=16, ctx=16384, k=32, capacity=64, headroom=8,
                         recall=16, cpu_frac=0.082),
    # configs[4]: batch 64 on 8 GPUs = 8 per GPU, 128K, top-128
    "qwen3-32b-128k": dict(layers=64, hq=64, hkv=8, batch=8, ctx=131072, k=128, capacity=128, headroom=16,
                           recall=16, cpu_frac=0.082),
    # configs[3] at ONE GPU (batch 128): only the kernel view fits 180 GB (--tier static; the resident
    # share = k - round(8.2% k) = 59 blocks per unit, 5 recall slots): 171 GB of pool + digests
    "qwen3-32b-32k-b128": dict(layers=64, hq=64, hkv=8, batch=128, ctx=32768, k=64, capacity=59, headroom=5,
                               recall=16, cpu_frac=0.082, static_only=True),
    # configs[0]: 1 request, 1 layer, 32 Q / 8 KV heads, 4K context, top-32, fp32 KV: the C-ABI path
    # (scout_score_topk_split + scout_sparse_decode with a CPU partial merged), no engine
    "toy-4k-f32": dict(layers=1, hq=32, hkv=8, batch=1, ctx=4096, k=32, capacity=64, headroom=0,
                       recall=0, cpu_frac=0.082, kv="f32"),
}


def log(*a):
    if int(os.environ.get("RANK", "0")) == 0:
        print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
        sm = [float(r[0]) for r in rows if len(r) >= 6 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 6 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows if len(r) >= 6 for j in range(4) if r[2 + j].strip() == "Active"})
        loaded = [s for s in sm if s > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# -------------------------------------------------------------- workload --
def _gen(dev, seed, request, salt):
    from paper_2603_27138_b200.sharding import request_seed

    g = torch.Generator(device=dev)
    g.manual_seed(request_seed(seed, request, salt))
    return g


class TierWorkload:
    """Device tier mode (--tier device): the full decode step of the reference
    (plan, select + mark, ticket application, attention + merge, append of the
    token's K/V with seal write-through and LRU eviction, periodic recall of
    predicted \\ resident blocks), all bookkeeping on the device (K5).

    Synthetic, random-init data of the named shape, generated per GLOBAL
    request id from one seed (so a rank's shard is a slice of the global
    workload, and any subset of requests can be rebuilt alone): K/V pool, bf16
    digests (lo <= hi), queries following a closed path (drift), CPU partials,
    the tokens' new K/V. The initial placement keeps each unit's selected
    blocks minus the CPU share (the paper's 8.2%) resident, filled to capacity."""

    def __init__(self, cfg, dev, seed, max_steps, requests, warm_slots=0, victim_cache=True, host_units=0,
                 warm_seed=True):
        """requests: a contiguous range of global request ids (this rank's
        shard). warm_slots: pool slots per (layer, unit) beyond capacity + the
        open block + one in-flight ticket; they start with the warm images of
        the next-best blocks by the placement query (the victim cache, see
        scout_tier_layer) and keep evicted blocks' images later (warm_seed=False:
        they start empty and fill only with evictions). host_units:
        units of the global workload (the host tier's index space, shared by
        every rank's shard; 0 = this shard's)."""
        from paper_2603_27138_b200 import ops
        from paper_2603_27138_b200.engine import LayerState
        from paper_2603_27138_b200.tier import DeviceTieredCache

        self.cfg, self.dev, self.requests = cfg, dev, list(requests)
        assert self.requests == list(range(self.requests[0], self.requests[0] + len(self.requests))), \
            "a shard is a contiguous request range"
        L, hq, hkv = cfg["layers"], cfg["hq"], cfg["hkv"]
        B = len(self.requests)
        G = hq // hkv
        U = B * hkv
        nb = cfg["ctx"] // BS
        nbs = ((nb + (max_steps + BS - 1) // BS + 1 + 7) // 8) * 8  # room for the appended tokens
        k, cap = cfg["k"], cfg["capacity"]
        self.L, self.U, self.G, self.nb, self.k, self.B, self.hkv = L, U, G, nb, k, B, hkv
        self.host_units, self.host_unit0 = int(host_units) or U, self.requests[0] * hkv
        kv_dt = torch.bfloat16
        W = max(0, min(int(warm_slots), nb - cap)) if victim_cache else 0
        self.warm_slots, self.victim_cache, self.warm_seed = W, bool(victim_cache), bool(warm_seed)
        # pool slots per (layer, unit): every block for the pinned layer 0; else the
        # capacity's sealed fast blocks + the open block + one recall ticket in
        # flight (at most k blocks: predicted \ residency), so a unit can never
        # run out of slots, however far its selection drifted since the last recall,
        # + W slots of warm images (device victim cache)
        spu = [nbs] + [cap + 1 + k + W] * (L - 1)
        self.tier = DeviceTieredCache(L, U, nbs, capacity=cap, slots_per_unit=spu, device=dev,
                                      victim_cache=victim_cache)
        self.tier.pin_layer(0)
        self.pool = ops.alloc_pool(self.tier.n_slots, kv_dt, dev)
        sb = ops.slot_bytes(kv_dt)
        # host tier: the slow copy of every block. Synthetic and bounded: block
        # (layer, global unit, id) is image ((layer*host_units + unit)*nbs + id) % host_blocks,
        # the same on every rank; the device holds the same bytes for its fast
        # and warm blocks (one content per block whichever side reads it)
        self.host_blocks = 8192
        self.host_tier = torch.empty(self.host_blocks * sb, dtype=torch.uint8).pin_memory()
        self.host_tier.view(torch.bfloat16).normal_(generator=torch.Generator().manual_seed(seed))
        host_dev = self.host_tier.to(dev)
        # requests differ in length (by < one block), so seals (and their
        # write-through) spread over steps instead of all units at once
        lens = cfg["ctx"] - 2 * (torch.tensor(self.requests, dtype=torch.int32, device=dev) % 32)
        self.n_tokens = lens.repeat_interleave(hkv).contiguous()
        # decode drift: the queries move along a closed loop, one point per step
        # (n_path points, all precomputed in HBM), so selections change a little
        # every step and the CPU share settles where recalls balance it
        n_path = cfg.get("drift_points", 32)
        radius = cfg.get("drift", 0.0)
        per = hkv * G
        q0, du, dv, noise = (torch.empty(L, U * G, D, device=dev) for _ in range(4))
        self.cpu_o = torch.empty(L, U * G, D, device=dev)
        m, l_ = torch.empty(L, U * G, device=dev), torch.empty(L, U * G, device=dev)
        self.k_new, self.v_new = torch.empty(L, U, D, device=dev), torch.empty(L, U, D, device=dev)
        for i, r in enumerate(self.requests):
            g = _gen(dev, seed, r, 1)
            sl = slice(i * per, (i + 1) * per)
            for t in (q0, du, dv, noise, self.cpu_o):
                t[:, sl] = torch.randn(L, per, D, generator=g, device=dev)
            m[:, sl] = torch.randn(L, per, generator=g, device=dev)
            l_[:, sl] = torch.rand(L, per, generator=g, device=dev) * 40 + 1
            self.k_new[:, i * hkv:(i + 1) * hkv] = torch.randn(L, hkv, D, generator=g, device=dev)
            self.v_new[:, i * hkv:(i + 1) * hkv] = torch.randn(L, hkv, D, generator=g, device=dev)
        self.q_path_t, self.q_path_p = [], []
        for j in range(n_path if radius > 0 else 1):
            th = 2 * math.pi * j / n_path
            qt = q0 + radius * (math.cos(th) * du + math.sin(th) * dv)
            qp = qt + 0.33 * noise
            qp = qp * (qt.norm(dim=-1, keepdim=True) / qp.norm(dim=-1, keepdim=True))
            self.q_path_t.append(qt.to(cfg["q_dtype"]))
            self.q_path_p.append(qp.to(cfg["q_dtype"]))
        del q0, du, dv, noise
        self.q_true, self.q_pred = self.q_path_t[0], self.q_path_p[0]
        self.cpu_o = self.cpu_o.to(cfg.get("cpu_dtype", torch.float32))
        self.cpu_ml = torch.stack([m, l_], dim=-1).contiguous()
        self.out_o = torch.empty(L, U * G, D, device=dev)
        self.out_ml = torch.empty(L, U * G, 2, device=dev)
        cpu_per_unit = int(round(cfg["cpu_frac"] * k))
        uid = torch.arange(U, device=dev, dtype=torch.int64)[:, None]
        ids = torch.arange(nbs, device=dev, dtype=torch.int32)[None]
        layers = []
        self.warm_blocks = 0
        for li in range(L):
            dig = torch.empty(U, 2, D, nbs, dtype=kv_dt, device=dev)
            for i, r in enumerate(self.requests):
                g = _gen(dev, seed, r, 2000 + li)
                a = torch.randn(hkv, D, nbs, generator=g, device=dev).to(kv_dt)
                b = torch.randn(hkv, D, nbs, generator=g, device=dev).to(kv_dt)
                dig[i * hkv:(i + 1) * hkv, 0] = torch.minimum(a, b)
                dig[i * hkv:(i + 1) * hkv, 1] = torch.maximum(a, b)
            dig[..., nb:] = 0  # blocks still to be appended
            base = self.tier.layer_base[li] + torch.arange(U, device=dev, dtype=torch.int32)[:, None] * spu[li]
            warm = warm_rank = None
            if li == 0:  # pinned: every block resident
                table = torch.where(ids < nb, base + ids, -1)
            else:
                r_ = ops.score_topk_split(self.q_pred[li], dig, self.n_tokens, k, G)
                sel = r_["sel_ids"][:, :k].long()
                score = torch.empty(U, nbs, device=dev)
                drop = torch.empty(U, cpu_per_unit, dtype=torch.long, device=dev)
                for i, r in enumerate(self.requests):
                    g = _gen(dev, seed, r, 3000 + li)
                    score[i * hkv:(i + 1) * hkv] = torch.rand(hkv, nbs, generator=g, device=dev)
                    drop[i * hkv:(i + 1) * hkv] = torch.rand(hkv, k, generator=g, device=dev).argsort(dim=1)[:, :cpu_per_unit]
                score[:, nb:] = -1
                score.scatter_(1, sel, 2.0)
                score.scatter_(1, torch.gather(sel, 1, drop), -0.5)
                score[self.n_tokens % BS != 0, nb - 1] = 3.0  # an open block is always fast (kv_store.hpp:60-63)
                keep = score.argsort(dim=1, descending=True)[:, :cap]
                table = torch.full((U, nbs), -1, dtype=torch.int32, device=dev)
                table.scatter_(1, keep, (base + torch.arange(cap, device=dev, dtype=torch.int32)[None]).to(torch.int32))
                if W > 0 and warm_seed:
                    # warm images: the W best slow sealed blocks by the placement query's
                    # stacked digest score (what a prefill that ends with the whole KV in
                    # HBM can leave behind), in the slots after the fast ones; the worst
                    # of them is reused first
                    qs = self.q_pred[li].float().view(U, G, D)
                    lo, hi = dig[:, 0].float(), dig[:, 1].float()  # [U][D][nbs]
                    real = torch.zeros(U, nbs, device=dev)
                    for g_ in range(G):
                        qg = qs[:, g_, :, None]
                        real += torch.maximum(qg * lo, qg * hi).sum(1)
                    real[table >= 0] = -math.inf
                    real[:, nb:] = -math.inf
                    real[(self.n_tokens % BS != 0), nb - 1] = -math.inf  # the open block is fast
                    wid = real.argsort(dim=1, descending=True)[:, :W]  # best first
                    warm = torch.full((U, nbs), -1, dtype=torch.int32, device=dev)
                    warm.scatter_(1, wid, (base + cap + torch.arange(W, device=dev, dtype=torch.int32)[None]))
                    warm_rank = torch.zeros(U, nbs, dtype=torch.int64, device=dev)
                    warm_rank.scatter_(1, wid, W - 1 - torch.arange(W, device=dev, dtype=torch.int64)[None].expand(U, W))
                    del lo, hi, real
            # device content of the fast (and warm) blocks = their host-tier images
            for t in (table, warm):
                if t is None:
                    continue
                uu, bb = (t >= 0).nonzero(as_tuple=True)
                src = ((li * self.host_units + self.host_unit0 + uu.long()) * nbs + bb.long()) % self.host_blocks
                ops.recall_gather(self.pool, kv_dt, host_dev, src, t[uu, bb])
            if warm is not None:
                self.warm_blocks += int((warm >= 0).sum())
            self.tier.adopt(li, table.contiguous(), self.n_tokens, warm=warm, warm_rank=warm_rank)
            layers.append(LayerState(dig, torch.full((U, nbs), -1, dtype=torch.int32, device=dev)))
        del host_dev
        self.layer_states = layers
        self.cpu_per_unit = cpu_per_unit
        self.digest_bytes_layer = U * 2 * D * nb * 2
        self.engine = None

    @staticmethod
    def auto_warm_slots(cfg, batch, max_steps, dev, reserve_gib=12.0):
        """Warm slots per (layer, unit) that fill the HBM left after the pinned
        layer, the digests, the query paths and a reserve for the engine and
        the verification (the pool is sized for 180 GB of HBM3e)."""
        free, _ = torch.cuda.mem_get_info(dev)
        L, hkv, G = cfg["layers"], cfg["hkv"], cfg["hq"] // cfg["hkv"]
        U = batch * hkv
        nb = cfg["ctx"] // BS
        nbs = ((nb + (max_steps + BS - 1) // BS + 1 + 7) // 8) * 8
        qb = 2 if cfg["q_dtype"] == torch.bfloat16 else 4
        fixed = (L * U * 2 * D * nbs * 2 + U * nbs * 32768
                 + 2 * cfg.get("drift_points", 32) * L * U * G * D * qb + reserve_gib * 2**30)
        per_slot = (L - 1) * U * 32768
        spu = int((free - fixed) // per_slot)
        return max(0, min(spu - (cfg["capacity"] + 1 + cfg["k"]), nb - cfg["capacity"]))

    def make_engine(self, **kw):
        """(Re)create the engine over this workload's state (the tier state and
        token counts carry over; an old engine is closed first)."""
        from paper_2603_27138_b200.engine import DecodeEngine

        if self.engine is not None:
            self.engine.close()
        cfg = self.cfg
        opts = dict(recall_interval=cfg["recall"], recall_intervals=cfg.get("recall_intervals"),
                    recall_stagger=cfg.get("recall_policy") == "stagger",
                    cpu_dtype=cfg.get("cpu_dtype", torch.float32), recall_mode=cfg.get("recall_mode", 1),
                    host_units=self.host_units, host_unit0=self.host_unit0)
        opts.update(kw)
        self.engine = DecodeEngine(layers=self.L, batch=self.B, hq=cfg["hq"], hkv=cfg["hkv"], k=self.k,
                                   n_tokens=self.n_tokens, pool=self.pool, kv_dtype=torch.bfloat16,
                                   layer_states=self.layer_states, scale=1.0 / math.sqrt(D),
                                   host_tier=self.host_tier, q_dtype=cfg["q_dtype"], tier=self.tier,
                                   host_blocks=self.host_blocks, host_staging=True, **opts)
        return self.engine

    def step(self, s):
        j = s % len(self.q_path_t)
        self.engine.decode_step_kv(s, self.q_path_t[j], self.q_path_p[j], self.cpu_o, self.cpu_ml, self.k_new,
                                   self.v_new, self.out_o, self.out_ml)

    def k2_bytes(self, res_tokens_total):
        """Algorithmic bytes of one K2 launch: resident selected K+V rows, q in,
        CPU partial in, output out."""
        UG = self.U * self.G
        qb, cb = self.q_path_t[0].element_size(), self.cpu_o.element_size()
        return res_tokens_total * 2 * D * 2 + UG * (D * qb + (D * cb + 8) + (D + 2) * 4)


class StaticWorkload:
    """--tier static: the kernel view. Residency fixed at the paper's 8.2% CPU
    share (all but round(8.2% k) of each unit's selected blocks resident,
    filled to capacity), no appends, no recalls: K1 + K2 over a fixed split,
    the kernel view of the metric (the device tier mode carries the recall).
    Same synthetic data kinds as TierWorkload (one generator per rank)."""

    def __init__(self, cfg, dev, seed):
        from paper_2603_27138_b200 import ops
        from paper_2603_27138_b200.engine import DecodeEngine, LayerState

        self.cfg = cfg
        L, hq, hkv, B = cfg["layers"], cfg["hq"], cfg["hkv"], cfg["batch"]
        G = hq // hkv
        U = B * hkv
        nb = cfg["ctx"] // BS
        nbs = ((nb + 7) // 8) * 8
        k = cfg["k"]
        cap, head = cfg["capacity"], cfg["headroom"]
        self.L, self.U, self.G, self.nb, self.k = L, U, G, nb, k
        g = torch.Generator(device=dev)
        g.manual_seed(seed)
        gcpu = torch.Generator().manual_seed(seed)
        kv_dt = torch.bfloat16
        n_slots = U * nb + (L - 1) * U * (cap + head)
        pool = ops.alloc_pool(n_slots, kv_dt, dev)
        pv = pool.view(torch.bfloat16)
        for s in range(0, pv.numel(), 1 << 28):
            pv[s:min(pv.numel(), s + (1 << 28))].normal_(generator=g)
        self.pool = pool
        self.n_tokens = torch.full((U,), cfg["ctx"], dtype=torch.int32, device=dev)
        self.q_true = torch.randn(L, U * G, D, generator=g, device=dev)
        noise = torch.randn(L, U * G, D, generator=g, device=dev)
        qp = self.q_true + 0.33 * noise
        self.q_pred = qp * (self.q_true.norm(dim=-1, keepdim=True) / qp.norm(dim=-1, keepdim=True))
        self.q_true, self.q_pred = self.q_true.to(cfg["q_dtype"]), self.q_pred.to(cfg["q_dtype"])
        self.q_path_t, self.q_path_p = [self.q_true], [self.q_pred]
        self.cpu_o = torch.randn(L, U * G, D, generator=g, device=dev).to(cfg.get("cpu_dtype", torch.float32))
        m = torch.randn(L, U * G, generator=g, device=dev)
        l_ = torch.rand(L, U * G, generator=g, device=dev) * 40 + 1
        self.cpu_ml = torch.stack([m, l_], dim=-1).contiguous()
        self.out_o = torch.empty(L, U * G, D, device=dev)
        self.out_ml = torch.empty(L, U * G, 2, device=dev)
        layers = []
        host_blocks = 4096
        sb = ops.slot_bytes(kv_dt)
        self.host_tier = torch.empty(host_blocks * sb, dtype=torch.uint8).pin_memory()
        self.host_tier.view(torch.bfloat16).normal_(generator=gcpu)
        slot_base = U * nb
        cpu_per_unit = int(round(cfg["cpu_frac"] * k))
        for li in range(L):
            a = torch.randn(U, D, nbs, generator=g, device=dev).to(kv_dt)
            b = torch.randn(U, D, nbs, generator=g, device=dev).to(kv_dt)
            dig = torch.stack([torch.minimum(a, b), torch.maximum(a, b)], dim=1).contiguous()
            del a, b
            if li == 0:
                ids = torch.arange(nbs, device=dev, dtype=torch.int32)[None]
                table = torch.where(ids < nb, torch.arange(U, device=dev, dtype=torch.int32)[:, None] * nb + ids, -1)
                layers.append(LayerState(dig, table.contiguous()))
                continue
            r = ops.score_topk_split(self.q_pred[li], dig, self.n_tokens, k, G)
            sel = r["sel_ids"][:, :k].long()
            score = torch.rand(U, nbs, generator=g, device=dev)
            score[:, nb:] = -1
            score.scatter_(1, sel, 2.0)
            drop = torch.rand(U, k, generator=g, device=dev).argsort(dim=1)[:, :cpu_per_unit]
            cpu_ids = torch.gather(sel, 1, drop)
            score.scatter_(1, cpu_ids, -0.5)
            keep = score.argsort(dim=1, descending=True)[:, :cap]
            base = slot_base + (li - 1) * U * (cap + head)
            slots = base + torch.arange(U, device=dev)[:, None] * (cap + head) + torch.arange(cap, device=dev)[None]
            table = torch.full((U, nbs), -1, dtype=torch.int32, device=dev)
            table.scatter_(1, keep, slots.to(torch.int32))
            nrc = min(cpu_per_unit, head)
            dst = base + torch.arange(U, device=dev)[:, None] * (cap + head) + cap + torch.arange(nrc, device=dev)[None]
            # each unit's plan is one contiguous run of host images (one copy-engine call)
            run0 = ((li * U + torch.arange(U, device=dev)[:, None]) * 2654435761) % (host_blocks - nrc)
            src = run0 + torch.arange(nrc, device=dev)[None]
            layers.append(LayerState(dig, table, src.reshape(-1).to(torch.int64).cpu().contiguous(),
                                     dst.reshape(-1).to(torch.int32).cpu().contiguous()))
        self.layer_states = layers
        self.engine = DecodeEngine(layers=L, batch=B, hq=hq, hkv=hkv, k=k, n_tokens=self.n_tokens, pool=pool,
                                   kv_dtype=kv_dt, layer_states=layers, scale=1.0 / math.sqrt(D),
                                   recall_interval=0, host_tier=self.host_tier, host_staging=True,
                                   q_dtype=cfg["q_dtype"], cpu_dtype=cfg.get("cpu_dtype", torch.float32),
                                   recall_stagger=cfg.get("static_recall_policy", "stagger") == "stagger",
                                   recall_mode=0)
        self.cpu_per_unit = cpu_per_unit
        self.digest_bytes_layer = U * 2 * D * nb * 2
        self.k_new = self.v_new = None

    def step(self, s):
        self.engine.decode_step(s, self.q_true, self.q_pred, self.cpu_o, self.cpu_ml, self.out_o, self.out_ml)

    def k2_bytes(self, res_tokens_total):
        UG = self.U * self.G
        qb, cb = self.q_true.element_size(), self.cpu_o.element_size()
        return res_tokens_total * 2 * D * 2 + UG * (D * qb + (D * cb + 8) + (D + 2) * 4)


# Test hooks for the N > 1 plumbing on a 1-GPU box: SCOUT_DIST_BACKEND=gloo
# (collectives on host tensors) and SCOUT_BENCH_ONE_GPU=1 (every rank on cuda:0).
# The product runs NCCL, one rank per GPU.
BACKEND = os.environ.get("SCOUT_DIST_BACKEND", "nccl")


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("SCOUT_BENCH_ONE_GPU") == "1":
        local = 0
    if ws > 1:
        import torch.distributed as dist

        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(BACKEND)
    return ws, rank, local


def coll_dev(dev):
    """Where collective tensors live: the GPU under NCCL, the host under gloo."""
    return dev if BACKEND == "nccl" else torch.device("cpu")


def max_over_ranks(x, ws, dev):
    from paper_2603_27138_b200.sharding import max_over_ranks as m

    return m(x, coll_dev(dev)) if ws > 1 else x


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def timed(fn, steps, dev, ws):
    """CUDA-event time of `steps` calls of fn, barrier + synchronize on both
    sides, max over ranks (ms per step)."""
    barrier(ws)
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(steps):
        fn(i)
    b.record()
    torch.cuda.synchronize(dev)
    barrier(ws)
    return max_over_ranks(a.elapsed_time(b), ws, dev) / steps


# ---------------------------------------------------------------- verify --
def verify_step(wl, step, n_units=8, layers=None):
    """Run one more step (device path, outside the timed region) and re-derive
    its outputs in float64 on the device for a sample of (layer, unit) pairs,
    from a snapshot of their state taken right before the step (digests,
    planning view, the K/V of every block that view counts as resident):
      * K1: the top-k set by the stacked digest_score rule (digest.hpp:62-118;
        ties to the lower id) from float64 scores; a set that differs only
        inside a float64 near-tie (k-th and (k+1)-th score within 1e-12 of the
        terms' magnitude) is counted, not failed (tests/ pin it bit-exact
        against the reference sum order);
      * the split against the planning view (engine.hpp:239-241);
      * K2+K3: partial_attention over the resident share + merge with the CPU
        partial + finalize (attention.hpp:73-122), within the bf16 bar (2e-2
        relative per head, 5e-3 on the log-sum-exp)."""
    from paper_2603_27138_b200 import ops

    eng, dev, L, U, G, k = wl.engine, wl.pool.device, wl.L, wl.U, wl.G, wl.k
    eng.sync()
    torch.cuda.synchronize(dev)
    layers = layers or sorted({0, 1, L // 2, L - 1})
    units = sorted({int(x) for x in np.linspace(0, U - 1, n_units)})
    tr = wl.tier
    ntok = wl.n_tokens.clone()
    snap = {}
    sb = ops.slot_bytes(torch.bfloat16)
    for l in layers:
        tick = step * L + l
        plan = torch.where((tr.tier[l] == 1) | ((tr.ready[l] >= 0) & (tr.ready[l] <= tick)), tr.table[l], -1)
        for u in units:
            slots = plan[u].clone()
            live = torch.nonzero(slots >= 0).flatten()
            img = wl.pool.view(-1, sb)[slots[live].long()].clone()  # [n][slot bytes]: a mini pool
            snap[(l, u)] = (wl.layer_states[l].digests[u].double().clone(), slots, live, img)
    j = step % len(wl.q_path_t)
    qt_all, qp_all = wl.q_path_t[j], wl.q_path_p[j]
    wl.step(step)
    eng.sync()
    torch.cuda.synchronize(dev)
    k1 = eng.k1_outputs()
    out_o, out_ml = wl.out_o, wl.out_ml
    n_ok = n_tie = n_bad = split_bad = 0
    worst, worst_lse, worst_at = 0.0, 0.0, None
    slot_mismatch = live_diff = 0
    scale = 1.0 / math.sqrt(D)
    for (l, u), (dig, slots, live, img) in snap.items():
        nt = int(ntok[u])
        nb = (nt + BS - 1) // BS
        q_sel = (qt_all[0] if l == 0 else qp_all[l])[u * G:(u + 1) * G].double()  # [G][D]
        # stacked score: sum over (c, g) of max(q_g[c] lo[c], q_g[c] hi[c]), float64
        lo, hi = dig[0, :, :nb], dig[1, :, :nb]  # [D][nb]
        terms = torch.maximum(q_sel[:, :, None] * lo[None], q_sel[:, :, None] * hi[None])  # [G][D][nb]
        sc = terms.sum(dim=(0, 1)).cpu()
        mag = float(terms.abs().sum(dim=(0, 1)).max())
        kk = min(k, nb)
        order = sorted(range(nb), key=lambda b: (-float(sc[b]), b))
        want = sorted(order[:kk])
        nr, nc = int(k1["n_res"][l, u]), int(k1["n_cpu"][l, u])
        res = k1["res_ids"][l, u, :nr].tolist()
        cpu = k1["cpu_ids"][l, u, :nc].tolist()
        got = sorted(res + cpu)
        if got == want:
            n_ok += 1
        elif kk < nb and abs(float(sc[order[kk - 1]] - sc[order[kk]])) <= 1e-12 * mag:
            n_tie += 1
        else:
            n_bad += 1
        planned = set(int(b) for b in torch.nonzero(slots >= 0).flatten().tolist())
        if set(res) != set(got) & planned or set(cpu) != set(got) - planned:
            split_bad += 1
        # attention over the snapshot's resident blocks (rows < the count at attention)
        pos = {int(b): i for i, b in enumerate(live.tolist())}
        sl, rr = [], []
        for b in res:
            rows = nt - (nb - 1) * BS if b == nb - 1 else BS
            sl += [pos[b]] * rows
            rr += list(range(rows))
        if sl:
            kr, vr = ops.kv_read_tokens(img.view(-1), torch.bfloat16, sl, rr)
            kr, vr = kr.double(), vr.double()
            # debug: the engine's own slots on the live pool
            rs = k1["res_slots"][l, u, :nr].tolist()
            plan_slots = [int(slots[b]) for b in res]
            if rs != plan_slots:
                slot_mismatch += 1
            sl2 = []
            for b, s_ in zip(res, rs):
                rows = nt - (nb - 1) * BS if b == nb - 1 else BS
                sl2 += [s_] * rows
            kr2, vr2 = ops.kv_read_tokens(wl.pool, torch.bfloat16, sl2, rr)
            if not (torch.equal(kr2.double(), kr) and torch.equal(vr2.double(), vr)):
                live_diff += 1
        qt = qt_all[l][u * G:(u + 1) * G].double()
        co = wl.cpu_o[l][u * G:(u + 1) * G].double()
        cm = wl.cpu_ml[l][u * G:(u + 1) * G].double()
        for g in range(G):
            mx, den, acc = -math.inf, 0.0, torch.zeros(D, dtype=torch.float64, device=dev)
            if sl:
                s = (kr @ qt[g]) * scale
                mx = float(s.max())
                p = torch.exp(s - mx)
                den = float(p.sum())
                acc = p @ vr
            cmx, cden = float(cm[g, 0]), float(cm[g, 1])
            if cden > 0:  # merge (attention.hpp:100-114), the CPU partial's o normalised
                M = max(mx, cmx)
                wa = math.exp(mx - M) if den > 0 else 0.0
                wb = math.exp(cmx - M)
                acc = acc * wa + co[g] * cden * wb
                den, mx = den * wa + cden * wb, M
            o = out_o[l][u * G + g].double()
            if den == 0:
                worst = max(worst, float(o.abs().max()))
                continue
            ref = acc / den
            e = float((o - ref).abs().max() / ref.abs().max())
            if e > worst:
                worst_at = (l, u, g, len(res), len(cpu), nt)
            worst = max(worst, e)
            ml = out_ml[l][u * G + g].double()
            worst_lse = max(worst_lse, abs(float(ml[0]) + math.log(float(ml[1])) - (mx + math.log(den))))
    ok = n_bad == 0 and split_bad == 0 and worst <= 2e-2 and worst_lse <= 5e-3
    return {"pass": bool(ok), "step": step, "layers": layers, "units": units,
            "topk_sets_exact": n_ok, "topk_sets_in_float64_near_tie": n_tie, "topk_sets_wrong": n_bad,
            "split_wrong": split_bad, "attention_max_rel_err": worst, "lse_max_abs_err": worst_lse,
            "worst_at_layer_unit_head": worst_at, "slot_mismatch": slot_mismatch, "live_diff": live_diff,
            "tolerance": {"attention_rel": 2e-2, "lse_abs": 5e-3},
            "reference": "torch float64 recomputation on the device from a pre-step snapshot (digest_score / "
                         "select_topk / split / partial_attention + merge + finalize); bit-exact top-k against the "
                         "reference sum order is pinned in tests/"}


def output_sums(wl, gb, ws, rank):
    """Per-request sums of the last step's outputs, gathered from every rank
    (indexed by global request id)."""
    from paper_2603_27138_b200.sharding import gather_per_request

    per = wl.hkv * wl.G
    mine = wl.out_o.view(wl.L, wl.B, per, D).double().sum(dim=(0, 2, 3))  # [B]
    return gather_per_request(mine.to(coll_dev(mine.device)), gb, ws, rank).cpu() if ws > 1 else mine.cpu()


def cross_rank_replay(cfg, args, ws, rank, dev, steps_done, seed, gb, allsum, warm, vc, warm_seed=True):
    """N > 1, after everything else (rank 0 has freed its own workload): rank 0
    rebuilds the LAST rank's shard of the global workload (same requests, same
    host-tier index space, same warm slots), replays steps 1..steps_done
    alone and compares that step's per-request output sums with what that
    rank produced."""
    from paper_2603_27138_b200.sharding import request_shard

    res = None
    if rank == 0:
        first, n = request_shard(gb, ws, ws - 1)
        sub = TierWorkload(cfg, dev, seed, max_steps=args.max_steps, requests=range(first, first + n),
                           warm_slots=warm, victim_cache=vc, host_units=gb * cfg["hkv"], warm_seed=warm_seed)
        sub.make_engine()
        for s_ in range(1, steps_done + 1):
            sub.step(s_)
        sub.engine.sync()
        torch.cuda.synchronize(dev)
        got = output_sums(sub, gb, 1, 0)
        want = allsum[first:first + n]
        rel = float(((got - want).abs() / want.abs().clamp_min(1e-30)).max())
        res = {"shard_recomputed": [first, first + n], "rank": ws - 1, "steps_replayed": steps_done,
               "max_rel_diff_of_output_sums": rel, "pass": rel <= 1e-3}
        sub.engine.close()
        del sub
    barrier(ws)
    return res


# ------------------------------------------------------------ CPU baseline --
class RefBaseline:
    """The reference's select_topk (stacked) + partial_attention + merge +
    finalize per (request, layer) on host cores, via oracle/_ref/libscout_ref.so
    (the unmodified reference headers). Inputs: a bounded sample of the same
    workload shape (S distinct (request, layer) inputs, cycled)."""

    def __init__(self, cfg, threads=None, sample_layers=4, seed=0):
        sys.path.insert(0, str(ROOT / "oracle"))
        import py_oracle as P

        self.ref = P.ref()
        self.cfg = cfg
        if self.ref is None:
            return
        hq, hkv, k = cfg["hq"], cfg["hkv"], cfg["k"]
        nb = cfg["ctx"] // BS
        G = hq // hkv
        self.threads = threads or os.cpu_count()
        rng = np.random.default_rng(seed)
        S = self.S = sample_layers
        q = rng.standard_normal((S, hq, D)).astype(np.float32).astype(np.float64)
        a = rng.standard_normal((S, hkv, D, nb)).astype(np.float32)
        b = rng.standard_normal((S, hkv, D, nb)).astype(np.float32)
        bf = lambda x: torch.from_numpy(x).bfloat16().double().numpy()  # noqa: E731
        dig = np.stack([bf(np.minimum(a, b)), bf(np.maximum(a, b))], axis=2)  # [S][hkv][2][D][nb]
        del a, b
        resident = np.zeros((S, hkv, nb), np.int32)
        res_index = np.zeros((S, hkv, nb), np.int32)
        cap = cfg["capacity"]
        ncpu = int(round(cfg["cpu_frac"] * k))
        for s_ in range(S):
            for u in range(hkv):
                ids, _ = P.unit_topk(q[s_, u * G:(u + 1) * G], dig[s_, u], nb, k)
                keep = [int(i) for i in rng.permutation(ids)[ncpu:]]
                chosen = set(int(i) for i in ids)
                others = [int(i) for i in rng.permutation(nb) if int(i) not in chosen][: cap - len(keep)]
                for j, bid in enumerate(sorted(keep + others)):
                    resident[s_, u, bid] = 1
                    res_index[s_, u, bid] = j
        kv = bf(rng.standard_normal((S, hkv, cap, 2, BS, D)).astype(np.float32))
        self._args = (S, hq, hkv, D, nb, k, np.ascontiguousarray(q), np.ascontiguousarray(dig), resident,
                      np.ascontiguousarray(kv), res_index, cap)
        self.sample = (f"(request, layer) units of the {cfg['layers']}-layer workload ({S} distinct inputs cycled): "
                       f"per unit {hkv} x [select_topk over {nb} stacked digests, split vs residency, {G} x "
                       f"partial_attention over the resident top-{k} share, merge with a pre-staged CPU partial, "
                       f"finalize]")
        t = self.run(self.threads)  # calibrate: one unit per thread
        self.units_per_s_est = self.threads / t

    def run(self, n):
        import ctypes as C

        chk = C.c_double()
        return self.ref.ref_cpu_baseline(*self._args, int(n), self.threads, C.byref(chk))

    def measure(self, seconds):
        n = max(self.threads, int(seconds * self.units_per_s_est))
        t = self.run(n)
        ups = n / t
        return dict(units_per_s=ups, tok_s=ups / self.cfg["layers"], seconds=t, units=n, threads=self.threads,
                    sample=f"{n} " + self.sample)


def measure_cpu_worker(wl, cfg, seconds=4.0):
    """The CPU co-attention worker (scout_cpu_partial_attention: AMX-BF16 tiles
    where the CPU has them, else AVX-512; all host threads) on this box over
    the workload's CPU share at the paper's 8.2%, standalone (the composed step
    runs it inside: e2e_with_cpu_worker)."""
    from paper_2603_27138_b200 import ops

    U, G = wl.U, wl.G
    nc = max(int(round(cfg["cpu_frac"] * cfg["k"])), 1)
    hb = wl.host_tier.numel() // ops.slot_bytes(torch.bfloat16)
    rng = np.random.default_rng(7)
    idx = torch.from_numpy(rng.integers(0, hb, size=(U, nc)).astype(np.int64))
    nb = torch.full((U,), nc, dtype=torch.int32)
    q = torch.randn(U * G, D)

    def rate(secs):
        ops.cpu_partial_attention(wl.host_tier, torch.bfloat16, idx, nb, q, G)  # warm
        n, t0 = 0, time.time()
        while time.time() - t0 < secs:
            ops.cpu_partial_attention(wl.host_tier, torch.bfloat16, idx, nb, q, G)
            n += 1
        return n * U * nc / (time.time() - t0)

    bps = rate(seconds)
    kernel = ops.cpu_coattn_kernel(torch.bfloat16)
    per_step = nc * U * (wl.L - 1)
    return {"blocks_per_s": bps, "threads": os.cpu_count(), "blocks_per_step_at_8.2pct": per_step,
            "ms_per_step_at_8.2pct": 1000.0 * per_step / bps, "gb_per_s": bps * ops.slot_bytes(torch.bfloat16) / 1e9,
            "kernel": f"scout_cpu_partial_attention (csrc/cpu_coattn.cpp, {kernel})"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------------- main --
def run_reference(args, cfg, ws, rank):
    if rank != 0:
        return
    rb = RefBaseline(cfg)
    if rb.ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libscout_ref.so not built"}), flush=True)
        return
    vals, units, r = [], [], None
    for i in range(args.warmup + args.steps):
        r = rb.measure(1.0)
        if i >= args.warmup:
            vals.append(r["tok_s"])
            units.append(r["units"])
    v = float(np.mean(vals))
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 * cfg["batch"] / v if v else None,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": args.config, "batch_per_gpu": cfg["batch"], "context": cfg["ctx"],
                       "layers": cfg["layers"], "heads": f"{cfg['hq']}q/{cfg['hkv']}kv", "top_k": cfg["k"],
                       "parallelism": "reference CPU (std::thread over all host cores), rank 0"},
            "timing": {"sampled": True, "units_per_whole_step": cfg["batch"] * cfg["layers"],
                       "units_timed_per_step": int(np.mean(units)),
                       "note": "each step times a ~1 s bounded sample of the step's (request, layer) units and "
                               "extrapolates: ms_per_step is the whole-step time at that rate, not wall time"},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": r["threads"], "kind": "reference",
                             "sample": "each step: " + r["sample"] + f"; {cpu_model()}"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


METRIC = "sparse decode-attn tokens/s/GPU at Qwen3-32B 32K; HBM GB/s vs peak"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64, help="timed steps (a multiple of 32: the drift loop)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="scout", choices=["scout", "reference"])
    ap.add_argument("--config", default="qwen3-32b-32k", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="requests per GPU (default: config; weak scaling)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="total requests split across ranks (strong scaling, e.g. config 4: 128)")
    ap.add_argument("--e2e-steps", type=int, default=64)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the cadence comparison and the CPU-worker e2e (faster)")
    ap.add_argument("--profile", action="store_true", help="short run for ncu: no e2e / baseline / extras")
    ap.add_argument("--tier", default="device", choices=["static", "device"],
                    help="device (default): the full decode step -- append + digest refresh, device tier "
                         "bookkeeping (LRU eviction, recall tickets), recalls (scout_engine_decode_step_kv); "
                         "static: residency fixed at the paper's 8.2%% CPU share, no appends (kernel view)")
    ap.add_argument("--drift", type=float, default=0.15,
                    help="device tier mode: radius of the closed query path the queries follow step by step "
                         "(0 = stationary)")
    ap.add_argument("--recall-policy", default="reference", choices=["reference", "stagger"],
                    help="reference (default): layer i is due when step - last_recall >= 16 "
                         "(recall.hpp:114-126), so every layer recalls at steps 16, 32, ...; stagger: layer i "
                         "recalls when (step + i) %% 16 == 0 (the same volume spread over the steps)")
    ap.add_argument("--recall-mode", default="sm", choices=["ce", "sm"],
                    help="recall copies: an SM gather kernel over the mapped host tier (sm, default) or the copy "
                         "engines, one cudaMemcpyAsync per contiguous run (ce)")
    ap.add_argument("--warm-slots", type=int, default=-1,
                    help="device tier mode: pool slots per (layer, unit) for warm images of slow blocks (the device "
                         "victim cache); -1 (default): fill the HBM left after the rest of the workload")
    ap.add_argument("--victim-cache", default="on", choices=["on", "off"],
                    help="off: every recall copies its blocks from the host tier (no warm images)")
    ap.add_argument("--warm-seed", default="on", choices=["on", "off"],
                    help="off: the warm slots start empty (no images left by the placement); only evicted "
                         "blocks' images fill them")
    ap.add_argument("--recall-calibrate", type=int, default=0,
                    help="device tier mode: profile this many recall-free steps first and calibrate per-layer "
                         "recall intervals from their CPU ratios (calibrate_intervals, recall.hpp:66-95, the "
                         "harness's calibrate command); 0 (default): every 16 steps, BASELINE's config")
    ap.add_argument("--beta", type=float, default=0.12, help="calibration threshold (EngineConfig::beta)")
    ap.add_argument("--q-dtype", default="bf16", choices=["bf16", "f32"],
                    help="query dtype (q_true / q_pred); bf16 = the model's projection output")
    ap.add_argument("--cpu-dtype", default="bf16", choices=["bf16", "f32"],
                    help="CPU-partial o as the host worker hands it over (bf16 halves the largest H2D stream)")
    ap.add_argument("--seed", type=int, default=1234)
    args = ap.parse_args()
    if args.profile:  # ncu replays kernels one at a time: no K1 beside a K2 that waits for it
        os.environ["SCOUT_K1K2_OVERLAP"] = "0"
    cfg = dict(CONFIGS[args.config])
    cfg["q_dtype"] = torch.bfloat16 if args.q_dtype == "bf16" else torch.float32
    cfg["cpu_dtype"] = torch.bfloat16 if args.cpu_dtype == "bf16" else torch.float32
    cfg["drift"] = args.drift
    cfg["recall_policy"] = args.recall_policy
    cfg["recall_mode"] = 1 if args.recall_mode == "sm" else 0
    if args.batch:
        cfg["batch"] = args.batch
    ws, rank, local = dist_setup()
    from paper_2603_27138_b200.sharding import request_shard

    scaling = "strong" if args.global_batch else "weak"
    gb = args.global_batch or cfg["batch"] * ws
    first, cfg["batch"] = request_shard(gb, ws, rank)
    if args.impl == "reference":
        run_reference(args, cfg, ws, rank)
        barrier(ws)
        return
    if cfg.get("kv") == "f32":
        run_c_abi_f32(args, cfg, ws, rank, gb)
        barrier(ws)
        return
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2603_27138_b200 import lib, ops

    lib()  # native library must be present: no fallback
    t0 = time.time()
    tier_mode = args.tier == "device" and not cfg.get("static_only")
    args.max_steps = args.warmup + 3 * args.steps + 2 * args.e2e_steps + 48
    if tier_mode:
        vc = args.victim_cache == "on"
        warm = args.warm_slots if args.warm_slots >= 0 else (
            TierWorkload.auto_warm_slots(cfg, cfg["batch"], args.max_steps, dev) if vc else 0)
        if ws > 1:  # every rank the same (the smallest shard's budget decides)
            t = torch.tensor([warm], dtype=torch.int64, device=coll_dev(dev))
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
            warm = int(t)
        wl = TierWorkload(cfg, dev, seed=args.seed, max_steps=args.max_steps,
                          requests=range(first, first + cfg["batch"]), warm_slots=warm, victim_cache=vc,
                          host_units=gb * cfg["hkv"], warm_seed=args.warm_seed == "on")
        wl.make_engine()
    else:
        wl = StaticWorkload(cfg, dev, seed=args.seed + rank)
    torch.cuda.synchronize(dev)
    log(f"workload ready in {time.time() - t0:.1f}s: pool {wl.pool.numel() / 2**30:.1f} GiB")
    step_no = 0

    def run_steps(n):
        nonlocal step_no
        for _ in range(n):
            step_no += 1
            wl.step(step_no)

    calibration = None
    if tier_mode and args.recall_calibrate > 0:
        # harness.hpp:464-476: a recall-free profiling run, one RatioTrace sample
        # per (layer, step) -- here the batch's CPU tokens over its budget -- then
        # calibrate_intervals(trace, beta) for the measured run
        from paper_2603_27138_b200.engine import calibrate_intervals

        wl.make_engine(recall_interval=0)
        cpu_tr, bud_tr = [], []
        for _ in range(args.recall_calibrate):
            step_no += 1
            wl.step(step_no)
            c_, b_ = wl.engine.cpu_tokens()
            cpu_tr.append(c_)
            bud_tr.append(b_)
        ivals = calibrate_intervals(np.array(cpu_tr).T, np.array(bud_tr).T, args.beta)
        if ws > 1:  # one schedule for every rank: the shortest interval of each layer
            t = torch.tensor(ivals, dtype=torch.int64, device=coll_dev(dev))
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MIN)
            ivals = [int(x) for x in t.tolist()]
        cfg["recall_intervals"] = ivals
        calibration = {"profiling_steps": args.recall_calibrate, "beta": args.beta, "intervals": ivals,
                       "mean_ratio": [float(np.mean(np.array(cpu_tr)[:, l] / np.array(bud_tr)[:, l]))
                                      for l in range(wl.L)]}
        wl.make_engine()
        log(f"calibrated recall intervals: {ivals}")
    run_steps(args.warmup)
    wl.engine.sync()
    torch.cuda.synchronize(dev)
    res_tok_layers = []
    if not tier_mode:  # resident token count per K2 launch (stationary across steps)
        for li in range(wl.L):
            st = wl.layer_states[li]
            q = wl.q_true[0] if li == 0 else wl.q_pred[li]
            r = ops.score_topk_split(q, st.digests, wl.n_tokens, wl.k, wl.G, block_table=st.table)
            res_tok_layers.append(int(r["res_tokens"].sum()))
    torch.cuda.synchronize(dev)
    eng = wl.engine
    eng.stats()  # reset counters
    if tier_mode:
        eng.recall_stats(reset=True)
    eng.overlap_stats(reset=True)
    eng.set_timing(True)
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" selects the timed launches

    def timed_step(i):
        nonlocal step_no
        step_no += 1
        wl.step(step_no)
        if i == args.steps - 1:
            eng.sync()

    ms_step = timed(timed_step, args.steps, dev, ws)
    torch.cuda.nvtx.range_pop()
    clk = clocks.stop()
    k2_each = eng.k2_times()
    k2_total, k2_n, launches = eng.stats()
    eng.set_timing(False)
    # steps whose K1 ran beside K2 (the overlapped step): their timed launch
    # is the pair, and its bytes are K2's plus K1's digest stream
    ov_steps, ov_sms = eng.overlap_stats(reset=True)
    tier_info = None
    if tier_mode:  # the residency evolves: bytes from the last timed step's K1 lists
        k1o = eng.k1_outputs()
        res_tok_layers = [int(x) for x in k1o["res_tokens"].sum(1).tolist()]
        cpu_tok = int(k1o["cpu_tokens"].sum())
        eng.check_state()  # no rejected ticket, no slot shortage, check_split held on every (layer, unit)
        rc_warm, rc_copy = eng.recall_stats()
        tier_info = {"mode": "device (scout_engine_decode_step_kv)", "resident_token_frac_last_step":
                     sum(res_tok_layers) / max(sum(res_tok_layers) + cpu_tok, 1),
                     "recall": {"blocks_per_step": (rc_warm + rc_copy) / args.steps,
                                "warm_blocks_per_step": rc_warm / args.steps,
                                "copied_blocks_per_step": rc_copy / args.steps,
                                "h2d_bytes_per_step": rc_copy * 32768 / args.steps,
                                "warm_frac": rc_warm / max(rc_warm + rc_copy, 1),
                                "victim_cache": wl.victim_cache, "warm_slots_per_unit": wl.warm_slots,
                                "warm_seeded_at_placement": wl.warm_seed,
                                "warm_images_at_placement": wl.warm_blocks,
                                "pool_gib": wl.pool.numel() / 2**30,
                                "note": "a recalled block whose image still sits in a free pool slot (evicted "
                                        "earlier, or left by the placement) takes that slot back: a tier flip "
                                        "with no bytes moved, as in the reference (kv_store.hpp:201-218); the "
                                        "others are copied from the pinned host tier by the SM gather (K4)"},
                     "tokens_at_end": int(wl.n_tokens[0]), "host_tier_blocks": wl.host_blocks,
                     "query_drift": cfg["drift"], "check_state": "ok (check_split on device, every layer and unit)",
                     "note": "queries follow a closed path (drift radius); the CPU share settles where the "
                             "periodic recalls balance the drift"}
    k2_avg = k2_total / max(k2_n, 1)
    tok_s = gb / (ms_step / 1000.0)
    # ---- roofline for K2 (dominant kernel): one persistent launch covers all layers of a step
    k2_bytes = float(sum(wl.k2_bytes(t) for t in res_tok_layers))
    peaks = {}
    try:
        peaks = json.load(open(ROOT / "MEASURED_PEAKS.json"))
    except OSError:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    traffic, traffic_src, k1_traffic = None, None, None
    try:  # dram read+write bytes per K2 (and K1) launch from the committed ncu --set full captures
        tj = json.load(open(ROOT / "profiles" / "k2_traffic.json"))
        traffic, traffic_src = tj["bytes_per_launch"], tj.get("source", "profiles/k2_traffic.json")
        k1_traffic = tj.get("k1_bytes_per_launch")
    except (OSError, KeyError, ValueError):
        pass
    k1_bytes = float(wl.L * wl.digest_bytes_layer)
    ov_frac = min(1.0, ov_steps / max(k2_n, 1))
    launch_bytes = k2_bytes + ov_frac * k1_bytes  # average over the timed launches
    achieved = launch_bytes / (k2_avg / 1000.0) / 1e9
    # the steady launches: K2 of a step that follows a recall burst waits inside
    # (layer by layer) for the burst's PCIe copies; the median launch is the
    # kernel's own streaming rate
    k2_med = float(np.median(k2_each)) if k2_each else k2_avg
    achieved_med = (k2_bytes + (k1_bytes if ov_frac >= 0.5 else 0.0)) / (k2_med / 1000.0) / 1e9
    step_bytes = k2_bytes + k1_bytes
    step_gbs = step_bytes / (ms_step / 1000.0) / 1e9
    k2_share = k2_total / (ms_step * args.steps) if ws == 1 else None
    log(f"step {ms_step:.3f} ms, {tok_s:.0f} tok/s, K2 avg {k2_avg * 1000:.1f} us ({achieved:.0f} GB/s), "
        f"step {step_gbs:.0f} GB/s, K2 share {k2_share}")
    # ---- verification (outside the timed region): float64 re-derivation of one step
    verify = None
    if tier_mode and not args.profile:
        step_no += 1
        verify = verify_step(wl, step_no)
        log(f"verify: {verify['pass']} (top-k {verify['topk_sets_exact']} exact, {verify['topk_sets_wrong']} wrong; "
            f"attention max rel err {verify['attention_max_rel_err']:.2e})")
    allsum, verify_step_no = None, step_no
    if tier_mode and ws > 1 and not args.profile:
        allsum = output_sums(wl, gb, ws, rank)
    extras = {}
    if tier_mode and not args.profile and not args.no_extras:
        # ---- the other recall cadence on the same workload (state carries over)
        other = "stagger" if args.recall_policy == "reference" else "reference"
        wl.make_engine(recall_stagger=other == "stagger")
        run_steps(5)
        wl.engine.sync()

        def ostep(i):
            nonlocal step_no
            step_no += 1
            wl.step(step_no)
            if i == args.steps - 1:
                wl.engine.sync()

        ms_o = timed(ostep, args.steps, dev, ws)
        extras["recall_cadence"] = {
            args.recall_policy: {"value": tok_s, "ms_per_step": ms_step},
            other: {"value": gb / (ms_o / 1000.0), "ms_per_step": ms_o},
            "note": "reference: step - last_recall >= 16 for every layer (recall.hpp:114-126), so all layers "
                    "recall in the same step and the next step waits for all of their PCIe copies; stagger: "
                    "layer i at (step + i) % 16 == 0, the same volume spread over 16 steps"}
        wl.make_engine()
        log(f"cadence: {extras['recall_cadence']}")
    # ---- layer by layer: a decoder's loop, layer i's inputs produced after layer i-1's attention
    if tier_mode and not args.profile and not args.no_extras:
        ms_lw = run_layerwise(wl, args.steps, dev, ws, step0=step_no)
        step_no += 5 + args.steps
        extras["value_layerwise"] = {
            "value": gb / (ms_lw / 1000.0), "ms_per_step": ms_lw, "recall_policy": args.recall_policy,
            "path": "scout_engine_decode_layer per layer (C ABI): layer i's q_true / q_pred[i+1] written by a kernel "
                    "queued after layer i-1's attention (a decoder's data dependency), then begin_layer tickets, K1 "
                    "of layer i+1 on the engine stream beside K2 of layer i, one K2 launch per layer, post per layer"}
        log(f"layerwise {ms_lw:.3f} ms/step")
        if cfg.get("hidden"):
            ms_lq, rfrac = run_layerwise_qpred(wl, args.steps, dev, ws, step0=step_no)
            step_no += 5 + args.steps
            extras["value_layerwise_qpred"] = {
                "value": gb / (ms_lq / 1000.0), "ms_per_step": ms_lq, "resident_token_frac_last_step": rfrac,
                "path": "scout_engine_decode_layer_x per layer: K6 (tcgen05 GEMM, predict_next_query of the "
                        "model's hidden state, engine.hpp:237) makes q_pred of layer i+1 inside the engine, then K1 "
                        "of layer i+1 beside K2 of layer i; hidden %d, W_Q random-init (4 distinct, cycled)"
                        % cfg["hidden"]}
            log(f"layerwise with q prediction {ms_lq:.3f} ms/step")
    # ---- e2e through host buffers (pre-staged CPU partials)
    e2e = None
    if not args.profile:
        e2e = run_e2e(wl, args.e2e_steps, dev, ws, gb, tier_mode, step0=step_no)
        step_no += 5 + args.e2e_steps
        log(f"e2e {e2e['ms_per_step']:.3f} ms/step")
    e2e_worker = None
    if tier_mode and not args.profile and not args.no_extras:
        e2e_worker = run_e2e_worker(wl, args.e2e_steps, dev, ws, gb, step0=step_no)
        step_no += 5 + args.e2e_steps
        log(f"e2e with CPU worker {e2e_worker['ms_per_step']:.3f} ms/step")
    # ---- the same cadence with every recalled block copied over PCIe (no warm images)
    if tier_mode and not args.profile and not args.no_extras and wl.victim_cache:
        wl.tier.victim_cache = False
        wl.make_engine()
        run_steps(5)
        wl.engine.sync()
        wl.engine.recall_stats(reset=True)

        def vstep(i):
            nonlocal step_no
            step_no += 1
            wl.step(step_no)
            if i == args.steps - 1:
                wl.engine.sync()

        ms_v = timed(vstep, args.steps, dev, ws)
        w_, c_ = wl.engine.recall_stats()
        extras["victim_cache_off"] = {
            "value": gb / (ms_v / 1000.0), "ms_per_step": ms_v, "recall_policy": args.recall_policy,
            "copied_blocks_per_step": c_ / args.steps, "h2d_bytes_per_step": c_ * 32768 / args.steps,
            "note": "same workload and cadence, every recalled block copied from the host tier (PCIe)"}
        log(f"victim cache off: {ms_v:.3f} ms/step, {c_ / args.steps:.0f} copied blocks per step")
        wl.tier.forget_warm()
        wl.tier.victim_cache = True
        wl.make_engine()
    # ---- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.profile:
        rb = RefBaseline(cfg)
        r = rb.measure(12.0) if rb.ref is not None else None
        if r is not None:
            cpu = {"value": r["tok_s"], "unit": "tokens/s", "cores": r["threads"], "kind": "reference",
                   "sample": r["sample"] + f"; {cpu_model()}"}
    cpu_worker = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.profile:
        cpu_worker = measure_cpu_worker(wl, cfg)
    cpu_per_unit = wl.cpu_per_unit
    if allsum is not None:  # N > 1: rank 0 replays the last rank's shard alone (its own workload freed first)
        vc_, warm_, seed_ = wl.victim_cache, wl.warm_slots, wl.warm_seed
        wl.engine.close()
        wl = eng = None
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        verify["cross_rank"] = cross_rank_replay(cfg, args, ws, rank, dev, verify_step_no, args.seed, gb, allsum,
                                                 warm_, vc_, seed_)
    if rank == 0:
        line = {
            "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init KV, digests, queries, CPU partials; one seeded global workload, "
                    "generated per request)",
            "config": {"workload": args.config, "attention_shape": "Qwen3-32B" if cfg["hq"] == 64 else "Qwen3-8B",
                       "batch_per_gpu": cfg["batch"], "global_batch": gb, "context": cfg["ctx"],
                       "layers": cfg["layers"], "heads": f"{cfg['hq']}q/{cfg['hkv']}kv", "head_dim": D,
                       "block": BS, "top_k": cfg["k"], "q_dtype": args.q_dtype, "cpu_partial_dtype": args.cpu_dtype,
                       "gpu_cache_blocks_per_unit": cfg["capacity"],
                       "cpu_blocks_per_unit_at_placement": cpu_per_unit, "recall_every": cfg["recall"],
                       "recall_policy": args.recall_policy if tier_mode else "none (static view: fixed residency)",
                       "tier": args.tier,
                       "parallelism": f"request-sharded x{ws}, no collective",
                       "l2": "inputs larger than L2 (step working set %.1f GiB)" % (step_bytes / 2**30)},
            "step_gbs": step_gbs,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": (traffic + ov_frac * k1_traffic) if (traffic and k1_traffic) else traffic,
                         "traffic_source": traffic_src,
                         "kernel": ("sparse_decode_tc_kernel (K2+K3, one persistent launch per step = all layers)"
                                    if ov_frac == 0 else
                                    f"sparse_decode_tc_kernel (K2+K3, all layers) with score_topk_kernel (K1, all "
                                    f"layers) beside it on {ov_sms} SMs in {ov_steps} of {k2_n} timed steps (the "
                                    f"overlapped step): the timed launch is the pair, its bytes K2's + K1's"),
                         "bytes_per_launch": launch_bytes, "k2_bytes_per_step": k2_bytes,
                         "k1_bytes_per_step": k1_bytes, "overlapped_steps": ov_steps,
                         "avg_launch_us": k2_avg * 1000.0,
                         "median_launch_us": k2_med * 1000.0, "achieved_median": achieved_med,
                         "frac_median": achieved_med / peak, "launches_timed": len(k2_each),
                         "max_launch_us": max(k2_each) * 1000.0 if k2_each else None,
                         "avg_vs_median": "avg includes the steps after a recall burst, whose K2 waits "
                                          "layer by layer for the burst's PCIe copies (ready at the next "
                                          "step, kv_store.hpp:190-193); the median is the kernel streaming",
                         "share_of_step": k2_share, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy)",
                         # K2 only reads: the copy peak counts read+write bytes of a copy, so a
                         # read-dominated gather can exceed it; the read-only bulk-copy stream
                         # and 32 KiB random-gather ceilings measured on this hardware
                         # (profiles/r01_microbench.txt, r01_gather.txt) bound it tighter
                         "read_stream_gbs": 7400.0, "frac_of_read_stream": achieved / 7400.0,
                         "gather_32k_gbs": 6700.0, "frac_of_gather_32k": achieved / 6700.0},
            "clocks": clk,
            "gpu_launches": launches,
            "verify": verify,
            "tier": tier_info,
            "recall_calibration": calibration,
            "e2e": e2e,
            "e2e_with_cpu_worker": e2e_worker,
            **extras,
            "cpu_baseline": cpu,
            "cpu_coattention": cpu_worker,
        }
        print(json.dumps(line), flush=True)
    barrier(ws)


def run_c_abi_f32(args, cfg, ws, rank, gb):
    """BASELINE configs[0] (fp32 KV, one layer, 1 request): the engine's step
    (static residency, f32 KV) and, beside it, the C ABI called directly as a
    reference caller would bind it -- per step one scout_score_topk_split
    (stacked select_topk + split against the residency table) and one
    scout_sparse_decode (f32 CUDA-core path, merged with a CPU partial). The
    tier holds all but round(8.2% k) selected blocks. e2e: the query and CPU
    partial H2D and the output D2H around the step."""
    from paper_2603_27138_b200 import ops

    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    ops.slot_bytes(torch.float32)  # the native library must be present: no fallback
    hq, hkv, k = cfg["hq"], cfg["hkv"], cfg["k"]
    G, U = hq // hkv, cfg["batch"] * hkv
    nb = cfg["ctx"] // BS
    g = torch.Generator(device=dev).manual_seed(args.seed + rank)
    pool = ops.alloc_pool(U * nb, torch.float32, dev)
    pool.view(torch.float32).normal_(generator=g)
    dig = torch.randn(U, 2, D, nb, generator=g, device=dev)
    dig = torch.stack([dig.min(dim=1).values, dig.max(dim=1).values], dim=1).contiguous()
    n_tokens = torch.full((U,), cfg["ctx"], dtype=torch.int32, device=dev)
    q = torch.randn(U * G, D, generator=g, device=dev)
    r0 = ops.score_topk_split(q, dig, n_tokens, k, G)
    ncpu = int(round(cfg["cpu_frac"] * k))
    table = (torch.arange(U, device=dev, dtype=torch.int32)[:, None] * nb + torch.arange(nb, device=dev, dtype=torch.int32)[None]).contiguous()
    drop = torch.rand(U, k, generator=g, device=dev).argsort(dim=1)[:, :ncpu]
    table.scatter_(1, torch.gather(r0["sel_ids"].long(), 1, drop), -1)
    cpu_o = torch.randn(U * G, D, generator=g, device=dev)
    cpu_ml = torch.stack([torch.randn(U * G, generator=g, device=dev), torch.rand(U * G, generator=g, device=dev) + 1],
                         -1).contiguous()
    bufs, ws_ = {}, ops.DecodeWorkspace(U, G, dev)
    o = torch.empty(U * G, D, device=dev)
    ml = torch.empty(U * G, 2, device=dev)

    def step(qq, co, cm):
        r = ops.score_topk_split(qq, dig, n_tokens, k, G, block_table=table, out=bufs)
        ops.sparse_decode(qq, pool, torch.float32, r["res_slots"], r["res_ids"], r["n_res"], n_tokens, G, cpu_o=co,
                          cpu_ml=cm, o=o, ml=ml, workspace=ws_)

    for _ in range(args.warmup):
        step(q, cpu_o, cpu_ml)
    clocks = ClockSampler(local)
    clocks.start()
    ms = timed(lambda i: step(q, cpu_o, cpu_ml), args.steps, dev, ws)
    clk = clocks.stop()
    res_tok = int(bufs["res_tokens"].sum())
    nbytes = res_tok * 2 * D * 4 + U * 2 * D * nb * 4 + U * G * (D * 4 * 2 + 8 + (D + 2) * 4)
    # e2e: pinned host query + CPU partial in, output out, every step
    hq_, hco, hcm = q.cpu().pin_memory(), cpu_o.cpu().pin_memory(), cpu_ml.cpu().pin_memory()
    ho, hml = torch.empty(o.shape).pin_memory(), torch.empty(ml.shape).pin_memory()
    dq, dco, dcm = torch.empty_like(q), torch.empty_like(cpu_o), torch.empty_like(cpu_ml)

    def e2e_step(i):
        dq.copy_(hq_, non_blocking=True)
        dco.copy_(hco, non_blocking=True)
        dcm.copy_(hcm, non_blocking=True)
        step(dq, dco, dcm)
        ho.copy_(o, non_blocking=True)
        hml.copy_(ml, non_blocking=True)

    for i in range(args.warmup):
        e2e_step(i)
    ms_e2e_direct = timed(e2e_step, args.steps, dev, ws)
    ms_direct = ms
    # ---- the same step through the engine (static residency, f32 KV: K1 + the
    # per-layer f32 K2), device-resident and from pinned host buffers
    from paper_2603_27138_b200.engine import DecodeEngine, LayerState

    eng = DecodeEngine(layers=1, batch=cfg["batch"], hq=hq, hkv=hkv, k=k, n_tokens=n_tokens, pool=pool,
                       kv_dtype=torch.float32, layer_states=[LayerState(dig, table)], scale=1.0 / math.sqrt(D),
                       host_staging=True, q_dtype=torch.float32, cpu_dtype=torch.float32)
    q3, co3, cm3 = q[None].contiguous(), cpu_o[None].contiguous(), cpu_ml[None].contiguous()
    o3, ml3 = torch.empty(1, U * G, D, device=dev), torch.empty(1, U * G, 2, device=dev)
    hq3, hco3, hcm3 = q3.cpu().pin_memory(), co3.cpu().pin_memory(), cm3.cpu().pin_memory()
    ho3, hml3 = torch.empty(o3.shape).pin_memory(), torch.empty(ml3.shape).pin_memory()
    st_no = [0]

    def eng_step(i):
        st_no[0] += 1
        eng.decode_step(st_no[0], q3, q3, co3, cm3, o3, ml3)

    def eng_e2e(i):
        st_no[0] += 1
        eng.decode_step_host(st_no[0], hq3, hq3, hco3, hcm3, ho3, hml3)

    for i in range(args.warmup):
        eng_step(i)
    eng.sync()
    eng.stats()
    clocks = ClockSampler(local)
    clocks.start()
    ms = timed(eng_step, args.steps, dev, ws)
    clk = clocks.stop()
    launches = eng.stats()[2]
    for i in range(args.warmup):
        eng_e2e(i)
    eng.sync()
    ms_e2e = timed(eng_e2e, args.steps, dev, ws)
    ok = torch.equal(o3[0], o)  # the same kernels on the same inputs as the direct calls
    eng.close()
    peaks = {}
    try:
        peaks = json.load(open(ROOT / "MEASURED_PEAKS.json"))
    except OSError:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    if rank == 0:
        line = {"metric": METRIC, "value": gb / (ms / 1000.0), "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (random-init f32 KV, digests, query)",
                "config": {"workload": args.config, "batch_per_gpu": cfg["batch"], "context": cfg["ctx"], "layers": 1,
                           "heads": f"{hq}q/{hkv}kv", "head_dim": D, "block": BS, "top_k": k,
                           "cpu_blocks_per_unit": ncpu, "kv_dtype": "f32",
                           "path": "the engine (scout_engine_decode_step, static residency, f32 KV: K1 + the "
                                   "per-layer f32 CUDA-core K2 merged with the CPU partial); e2e through "
                                   "scout_engine_decode_step_host",
                           "l2": "working set %.1f MiB: fits L2 (a latency-bound config)" % (nbytes / 2**20)},
                "roofline": {"bound": "latency (one request, one layer: 8 units)", "achieved": nbytes / ms / 1e6,
                             "peak": peak, "unit": "GB/s", "frac": nbytes / ms / 1e6 / peak,
                             "traffic": None, "kernel": "K1 + K2 (f32), step bytes / step time"},
                "clocks": clk, "gpu_launches": launches,
                "e2e": {"value": gb / (ms_e2e / 1000.0), "unit": "tokens/s", "ms_per_step": ms_e2e,
                        "h2d_bytes_per_step": int(2 * hq3.numel() * 4 + hco3.numel() * 4 + hcm3.numel() * 4),
                        "d2h_bytes_per_step": int(ho3.numel() * 4 + hml3.numel() * 4)},
                "engine_matches_direct_calls": bool(ok),
                "c_abi_direct": {"ms_per_step": ms_direct, "value": gb / (ms_direct / 1000.0),
                                 "e2e_ms_per_step": ms_e2e_direct,
                                 "path": "scout_score_topk_split + scout_sparse_decode called directly (torch "
                                         "copies for the e2e H2D / D2H)"}}
        print(json.dumps(line), flush=True)


def run_layerwise(wl, steps, dev, ws, step0, **engine_kw):
    """The step as a decoder drives it: one scout_engine_decode_layer call per
    layer, layer i's queries written into the live query buffers by a copy
    queued after layer i-1's call (in a model they come from layer i-1's
    output, so nothing of layer i can start earlier)."""
    eng = wl.make_engine(**engine_kw)
    L = wl.L
    qt_live = torch.empty_like(wl.q_path_t[0])
    qp_live = torch.empty_like(wl.q_path_p[0])

    def one(s):
        j = s % len(wl.q_path_t)
        for i in range(L):
            qt_live[i].copy_(wl.q_path_t[j][i])
            if i + 1 < L:
                qp_live[i + 1].copy_(wl.q_path_p[j][i + 1])
            eng.decode_layer(s, i, qt_live[i], qp_live[i + 1] if i + 1 < L else None, wl.cpu_o[i], wl.cpu_ml[i],
                             wl.k_new[i], wl.v_new[i], wl.out_o[i], wl.out_ml[i])

    for s in range(5):
        one(step0 + 1 + s)
    eng.sync()

    def tstep(i):
        one(step0 + 6 + i)
        if i == steps - 1:
            eng.sync()

    ms = timed(tstep, steps, dev, ws)
    eng.check_state()
    wl.make_engine()
    return ms


def run_layerwise_qpred(wl, steps, dev, ws, step0, n_weights=4):
    """Layer by layer with the layer-ahead prediction inside the engine
    (scout_engine_decode_layer_x: K6, the tcgen05 GEMM, makes q_pred of layer
    i+1 from the model's hidden state, engine.hpp:237): x_i [batch][hidden]
    follows a closed path like the queries, W_Q^{i+1} [hidden][Hq*128] bf16
    random-init, n_weights distinct matrices cycled over the layers (each
    84 MB at Qwen3-32B: every call streams its W from HBM)."""
    from paper_2603_27138_b200 import ops

    cfg = wl.cfg
    L, B, hidden = wl.L, wl.B, cfg["hidden"]
    n_out = cfg["hq"] * D
    g = torch.Generator(device=dev)
    g.manual_seed(99)
    wqs = [ops.QueryPredictor(torch.randn(hidden, n_out, generator=g, device=dev) / math.sqrt(hidden), B)
           for _ in range(n_weights)]
    x0, du, dv = (torch.randn(L, B, hidden, generator=g, device=dev) for _ in range(3))
    eng = wl.make_engine(hidden=hidden)
    qt_live = torch.empty_like(wl.q_path_t[0])
    radius, n_path = cfg.get("drift", 0.0), cfg.get("drift_points", 32)

    def one(s):
        j = s % len(wl.q_path_t)
        th = 2 * math.pi * (s % n_path) / n_path
        x = x0 + radius * (math.cos(th) * du + math.sin(th) * dv)
        for i in range(L):
            qt_live[i].copy_(wl.q_path_t[j][i])
            nxt = i + 1 < L
            eng.decode_layer_x(s, i, qt_live[i], x[i] if nxt else None, wqs[(i + 1) % n_weights] if nxt else None,
                               wl.cpu_o[i], wl.cpu_ml[i], wl.k_new[i], wl.v_new[i], wl.out_o[i], wl.out_ml[i])

    for s in range(5):
        one(step0 + 1 + s)
    eng.sync()

    def tstep(i):
        one(step0 + 6 + i)
        if i == steps - 1:
            eng.sync()

    ms = timed(tstep, steps, dev, ws)
    k1o = eng.k1_outputs()
    res, cpu = int(k1o["res_tokens"].sum()), int(k1o["cpu_tokens"].sum())
    eng.check_state()
    wl.make_engine()
    del wqs
    return ms, res / max(res + cpu, 1)


def _pinned_inputs(wl, tier_mode):
    n = len(wl.q_path_t)
    h_qt = [t.cpu().pin_memory() for t in wl.q_path_t]
    h_qp = [t.cpu().pin_memory() for t in wl.q_path_p]
    h_kv = [wl.k_new.cpu().pin_memory(), wl.v_new.cpu().pin_memory()] if tier_mode else []
    return n, h_qt, h_qp, h_kv


def run_e2e(wl, steps, dev, ws, global_batch, tier_mode, step0):
    """Same step through the C++ engine with pinned HOST inputs/outputs
    (scout_engine_decode_step_kv_host / _host): H2D of q_true / q_pred / CPU
    partials / the token's K/V in layer chunks on a copy stream, D2H of the
    attention output and of each layer's CPU-side block ids on another, all
    inside the timed region."""
    L = wl.L
    eng = wl.engine
    n, h_qt, h_qp, h_kv = _pinned_inputs(wl, tier_mode)
    h_co = wl.cpu_o.cpu().pin_memory()
    h_cm = wl.cpu_ml.cpu().pin_memory()
    h_out = torch.empty(wl.out_o.shape, dtype=torch.float32).pin_memory()
    h_oml = torch.empty(wl.out_ml.shape, dtype=torch.float32).pin_memory()
    h_cpu_ids = torch.empty(L, wl.U, wl.k, dtype=torch.int32).pin_memory()
    h_n_cpu = torch.empty(L, wl.U, dtype=torch.int32).pin_memory()

    def one(s):
        j = s % n
        if tier_mode:
            eng.decode_step_kv_host(s, h_qt[j], h_qp[j], h_co, h_cm, *h_kv, h_out, h_oml, h_cpu_ids, h_n_cpu)
        else:
            eng.decode_step_host(s, h_qt[j], h_qp[j], h_co, h_cm, h_out, h_oml, h_cpu_ids, h_n_cpu)

    warm = 5
    for s in range(warm):
        one(step0 + 1 + s)
    eng.sync()

    def tstep(i):
        one(step0 + 1 + warm + i)
        if i == steps - 1:
            eng.sync()

    ms = timed(tstep, steps, dev, ws)
    h2d_bytes = sum(x.numel() * x.element_size() for x in (h_qt[0], h_qp[0], h_co, h_cm, *h_kv))
    d2h_bytes = sum(x.numel() * x.element_size() for x in (h_out, h_oml, h_cpu_ids, h_n_cpu))
    return {"value": global_batch / (ms / 1000.0), "unit": "tokens/s", "ms_per_step": ms, "steps": steps,
            "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
            "verified_by": "tests/test_gpu_engine_tier.py::test_engine_tier_host_path_matches_device_path "
                           "(bit-exact against the device path, step by step)",
            "path": "C ABI scout_engine_decode_step_%s (csrc/engine.cpp), pinned host buffers, CPU partials "
                    "pre-staged" % ("kv_host" if tier_mode else "host")}


def run_e2e_worker(wl, steps, dev, ws, global_batch, step0, threads=0, chunk_layers=4):
    """The composed step (device tier mode, host buffers): the engine's own CPU
    worker computes each layer's CPU partial during the step from the ids K1
    selected in that step and the step's predicted queries, publishing layer
    chunks that the running K2 merges (engine.hpp:236-273). Nothing is
    pre-staged: the step waits for the host's CPU share."""
    L = wl.L
    eng = wl.make_engine(cpu_worker=True, chunk_layers=chunk_layers, cpu_threads=threads)
    n, h_qt, h_qp, h_kv = _pinned_inputs(wl, True)
    h_out = torch.empty(wl.out_o.shape, dtype=torch.float32).pin_memory()
    h_oml = torch.empty(wl.out_ml.shape, dtype=torch.float32).pin_memory()

    def one(s):
        j = s % n
        eng.decode_step_kv_host(s, h_qt[j], h_qp[j], None, None, *h_kv, h_out, h_oml)

    warm = 5
    for s in range(warm):
        one(step0 + 1 + s)
    eng.sync()
    eng.worker_stats()

    def tstep(i):
        one(step0 + 1 + warm + i)
        if i == steps - 1:
            eng.sync()

    ms = timed(tstep, steps, dev, ws)
    cpu_ms, nsteps = eng.worker_stats()
    k1o = eng.k1_outputs()
    cpu_blocks = int(k1o["n_cpu"].sum())
    eng.check_state()
    h2d_bytes = sum(x.numel() * x.element_size() for x in (h_qt[0], h_qp[0], *h_kv))
    d2h_bytes = sum(x.numel() * x.element_size() for x in (h_out, h_oml)) + L * wl.U * (wl.k + 1) * 4
    out = {"value": global_batch / (ms / 1000.0), "unit": "tokens/s", "ms_per_step": ms, "steps": steps,
           "cpu_worker_ms_per_step": cpu_ms / max(nsteps, 1), "cpu_blocks_last_step": cpu_blocks,
           "threads": threads or os.cpu_count(), "h2d_bytes_per_step": h2d_bytes, "d2h_bytes_per_step": d2h_bytes,
           "verified_by": "tests/test_gpu_engine_worker.py (every (step, layer, unit) against the reference's "
                          "recompute_layer_attention, harness.hpp:318-329)",
           "path": "C ABI scout_engine_decode_step_kv_host with cfg.cpu_worker (csrc/engine.cpp + cpu_coattn.cpp): "
                   "CPU partials computed in the step, published per 4-layer chunk to the running K2"}
    wl.make_engine()
    return out


if __name__ == "__main__":
    main()
