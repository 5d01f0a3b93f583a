"""K2 per-step time at a config under variations (recall off, layers, batch),
to separate per-layer fixed costs from streaming."""
import sys
import time

sys.path[:0] = ["."]
import torch

import bench

dev = torch.device("cuda")
for name, over in (("cfg2", {}), ("cfg2 no recall", {"recall": 0}), ("cfg2 L=12", {"layers": 12}),
                   ("cfg2 L=12 no recall", {"layers": 12, "recall": 0})):
    cfg = dict(bench.CONFIGS["qwen3-8b-16k"])
    cfg.update(over)
    cfg["q_dtype"] = torch.bfloat16
    wl = bench.Workload(cfg, dev, seed=1)
    eng = wl.engine
    for s in range(3):
        wl.step(s + 1)
    eng.sync()
    torch.cuda.synchronize()
    eng.stats()
    eng.set_timing(True)
    for s in range(20):
        wl.step(10 + s)
    eng.sync()
    torch.cuda.synchronize()
    k2, n, _ = eng.stats()
    eng.set_timing(False)
    print(f"{name}: K2 {k2 / n * 1000:.1f} us per launch ({cfg['layers']} layers: {k2 / n * 1000 / cfg['layers']:.1f} us/layer)",
          flush=True)
    del wl, eng
    torch.cuda.empty_cache()
