"""K6 at the Qwen3-32B shape (hidden 5120 -> 64 x 128 query features, batch
32): device time per predict_next_query call (CUDA graph of 20 calls, so
host launch cost is excluded) and the weight-streaming bandwidth
(algorithmic bytes = W + x + q_pred)."""
import json
import sys

sys.path[:0] = ["."]
import torch

from paper_2603_27138_b200 import ops

hidden, n_out, batch = 5120, 8192, 32
w = (torch.randn(hidden, n_out, device="cuda") / hidden ** 0.5).bfloat16()
x = torch.randn(batch, hidden, device="cuda")
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6537.0)
for ks in (0, 148, 296):
    qp = ops.QueryPredictor(w, batch, max_ctas=ks)
    o = torch.empty(batch, n_out, device="cuda")
    for _ in range(5):
        qp(x, out_f32=o)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            qp(x, out_f32=o)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 100 * 1000
    byts = hidden * n_out * 2 + batch * hidden * 4 + batch * n_out * 4
    print(f"max_ctas {ks}: {us:.1f} us per layer, {byts / us / 1e3:.0f} GB/s ({byts / us / 1e3 / peak:.2f} of {peak:.0f})")
