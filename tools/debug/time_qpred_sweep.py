import os
import subprocess
import sys
sys.path[:0] = ["."]
if len(sys.argv) == 1:
    for nst in ("", "2", "3", "4", "8"):
        for ks in (2, 4, 7, 9, 16):
            env = dict(os.environ)
            if nst:
                env["SCOUT_QP_NST"] = nst
            out = subprocess.run([sys.executable, __file__, str(ks)], env=env, capture_output=True, text=True).stdout
            print(f"nst {nst or 'auto'} ksplit {ks}: {out.strip()}", flush=True)
    sys.exit(0)
import torch
from paper_2603_27138_b200 import ops
hidden, n_out, batch, ks = 5120, 8192, 32, int(sys.argv[1])
w = (torch.randn(hidden, n_out, device="cuda") / hidden ** 0.5).bfloat16()
x = torch.randn(batch, hidden, device="cuda")
qp = ops.QueryPredictor(w, batch, ksplit=ks)
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
print(f"{us:.1f} us, {hidden * n_out * 2 / us / 1e3:.0f} GB/s")
