"""One K6 (q-prediction GEMM) launch at Qwen3-32B shape, for an ncu capture (round_check.sh)."""
import sys
sys.path[:0] = ["."]
import torch
from paper_2603_27138_b200 import ops
hidden, n_out, batch = 5120, 8192, 32
w = (torch.randn(hidden, n_out, device="cuda") / hidden ** 0.5).bfloat16()
x = torch.randn(batch, hidden, device="cuda")
qp = ops.QueryPredictor(w, batch, max_ctas=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
for _ in range(3):
    qp(x)
torch.cuda.synchronize()
