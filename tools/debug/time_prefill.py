"""scout_tier_prefill at the config-3 shape for one layer (256 units, 32K
tokens each, capacity 64 + 65 slots): device only, and with every sealed
block written through to a pinned host tier (the slow copy over PCIe)."""
import sys
sys.path[:0] = ["."]
import torch
from paper_2603_27138_b200 import ops
from paper_2603_27138_b200.tier import DeviceTieredCache

U, T, nbs, cap, spu = 256, 32768 - 30, 520, 64, 129
dev = torch.device("cuda")
kv = torch.bfloat16
k = torch.randn(U, T, 128, device=dev)
v = torch.randn(U, T, 128, device=dev)
nt = torch.full((U,), T, dtype=torch.int32)
sb = ops.slot_bytes(kv)
host = torch.empty(U * nbs * sb, dtype=torch.uint8).pin_memory()
for with_host in (False, True):
    times = []
    for r in range(3):
        tc = DeviceTieredCache(1, U, nbs, capacity=cap, slots_per_unit=spu)
        pool = ops.alloc_pool(tc.n_slots, kv)
        dig = torch.empty(U, 2, 128, nbs, dtype=kv, device=dev)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        tc.prefill(0, k, v, nt, pool, kv, dig, host_tier=host if with_host else None)
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        del tc, pool, dig
    ms = min(times)
    rows_gb = 2 * U * T * 128 * 4 / 1e9
    host_gb = U * (T // 64) * sb / 1e9
    print(f"prefill one layer ({U} units x {T} tokens), host write-through {with_host}: {ms:.2f} ms "
          f"(rows in {rows_gb:.1f} GB f32: {rows_gb / ms:.2f} TB/s; host images {host_gb:.1f} GB"
          f"{': %.1f GB/s' % (host_gb / ms * 1e3) if with_host else ''})", flush=True)
