"""K6 at the Qwen3-32B shape: time per predict_next_query launch and the
weight-streaming bandwidth (algorithmic bytes = W + x^ + q_pred)."""
import json
import sys

sys.path[:0] = ["."]
import torch

from paper_2603_27138_b200 import ops

hidden, n_out, batch = 5120, 8192, 32
w = (torch.randn(hidden, n_out, device="cuda") / hidden ** 0.5).bfloat16()
x = torch.randn(batch, hidden, device="cuda")
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6537.0)
for ks in (1, 2, 3, 4, 6):
    qp = ops.QueryPredictor(w, batch, ksplit=ks)
    for _ in range(5):
        qp(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 50
    for _ in range(n):
        qp(x)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1000
    byts = hidden * n_out * 2 + batch * hidden * 4 + batch * n_out * 4
    print(f"ksplit {ks}: {us:.1f} us per layer, {byts / us / 1e3:.0f} GB/s ({byts / us / 1e3 / peak:.2f} of {peak:.0f})")
