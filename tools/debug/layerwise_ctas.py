"""Layer-by-layer mode (scout_engine_decode_layer) at several K2 widths: the
SMs a single-layer K2 leaves free run K1 of the next layer beside it."""
import os, sys
sys.path[:0] = ["."]
import torch
import bench

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="reference")
dev = torch.device("cuda")
W = bench.TierWorkload.auto_warm_slots(cfg, 32, 900, dev)
wl = bench.TierWorkload(cfg, dev, 1234, 900, range(32), warm_slots=W)
wl.make_engine()
step = 0
for s in range(5):
    step += 1
    wl.step(step)
for ctas in [int(x) for x in (sys.argv[1:] or ["120", "112", "104", "96", "88", "80", "-1"])]:
    ms = bench.run_layerwise(wl, 32, dev, 1, step, layer_ctas=ctas)
    step += 5 + 32
    print(f"layer_ctas {ctas}: {ms:.3f} ms/step", flush=True)
