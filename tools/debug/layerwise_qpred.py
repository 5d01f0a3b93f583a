"""Layer by layer with K6 inside (bench.run_layerwise_qpred) and without, on
one config-3 workload; SCOUT_QP_NST / SCOUT_LW_K2_CTAS from the environment."""
import sys
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
for _ in range(5):
    step += 1
    wl.step(step)
for r in range(2):
    ms = bench.run_layerwise(wl, 32, dev, 1, step)
    step += 37
    msq, fr = bench.run_layerwise_qpred(wl, 32, dev, 1, step)
    step += 37
    print(f"layerwise {ms:.3f} ms, with K6 {msq:.3f} ms (resident frac {fr:.3f})", flush=True)
