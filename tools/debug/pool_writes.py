"""Debug: which resident blocks change during one tier-mode step (bench workload, small batch)."""
import sys
sys.path[:0] = ["."]
import torch
import bench
from paper_2603_27138_b200 import ops

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.0, recall_policy="reference", batch=4)
dev = torch.device("cuda")
wl = bench.TierWorkload(cfg, dev, 1234, 200, range(4))
wl.make_engine()
for s in range(1, 38):
    wl.step(s)
wl.engine.sync(); torch.cuda.synchronize()
sb = ops.slot_bytes(torch.bfloat16)
tr = wl.tier
L, U = wl.L, wl.U
# duplicate slots across the fast/in-flight tables and free stacks?
for l in range(L):
    used = tr.table[l][tr.table[l] >= 0]
    free = torch.tensor([x for u in range(U) for x in tr.free_ring(l, u)], dtype=torch.int32, device=used.device)
    both = torch.cat([used, free])
    if both.unique().numel() != both.numel():
        print("layer", l, "duplicate slots: table", used.numel(), "free", free.numel(), "unique", both.unique().numel())
pv = wl.pool.view(-1, sb)
snap = pv.clone()
wl.step(38)
wl.engine.sync(); torch.cuda.synchronize()
diff = (pv != snap).any(dim=1).nonzero().flatten()
print("slots changed:", diff.numel())
for s_ in diff[:20].tolist():
    # which (layer, unit, block) owns it?
    hit = (tr.table == s_).nonzero().tolist()
    rows = (pv[s_].view(2, 64 * 128 * 2) != snap[s_].view(2, -1)).view(2, -1, 2).any(-1)
    print("slot", s_, "owners", hit, "bytes changed", int((pv[s_] != snap[s_]).sum()))
