"""Per-unit vs per-block cost of the CPU co-attention worker: n units with b
blocks each (b = 0..16) over a 256 MB host tier, at 1 thread and all threads."""
import os, sys, time
sys.path[:0] = ["."]
import torch
from paper_2603_27138_b200 import ops

G, k = 8, 64
hb = 8192
sb = ops.slot_bytes(torch.bfloat16)
host = torch.empty(hb * sb, dtype=torch.uint8)
if torch.cuda.is_available():
    host = host.pin_memory()
host.view(torch.bfloat16).normal_()
print("kernel", ops.cpu_coattn_kernel(torch.bfloat16))
for T in (1, os.cpu_count()):
    n = 256 * (T if T > 1 else 1)
    for b in (0, 1, 2, 4, 8, 16):
        idx = torch.randint(0, hb, (n, k), dtype=torch.int64)
        nb = torch.full((n,), b, dtype=torch.int32)
        q = torch.randn(n * G, 128)
        ops.cpu_partial_attention(host, torch.bfloat16, idx, nb, q, G, threads=T)
        reps = 5
        t0 = time.perf_counter()
        for _ in range(reps):
            ops.cpu_partial_attention(host, torch.bfloat16, idx, nb, q, G, threads=T)
        t = (time.perf_counter() - t0) / reps
        print(f"threads {T:2d} blocks/unit {b:2d}: {t * 1e6 / n * T:7.2f} us per unit-thread, "
              f"{(t * 1e6 / (n * b) * T) if b else 0:6.2f} us per block-thread, {n * b / t / 1e6:.2f} M blocks/s", flush=True)
