"""Composed step (in-engine CPU worker): query / partial dtypes, and a per-chunk
profile (SCOUT_CW_PROF=1) of a few steps."""
import os, sys
sys.path[:0] = ["."]
import torch
import bench

dev = torch.device("cuda")
for qd, cd in [(torch.bfloat16, torch.bfloat16), (torch.float32, torch.float32)]:
    cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
    cfg.update(q_dtype=qd, cpu_dtype=cd, drift=0.15, recall_policy="reference")
    wl = bench.TierWorkload(cfg, dev, 1234, 400, range(32), warm_slots=0)
    wl.make_engine()
    for s in range(1, 21):
        wl.step(s)
    r = bench.run_e2e_worker(wl, 16, dev, 1, 32, 20)
    print(f"q {qd} partials {cd}: {r['ms_per_step']:.2f} ms/step, worker {r['cpu_worker_ms_per_step']:.2f} ms, "
          f"{r['cpu_blocks_last_step']} blocks", flush=True)
    wl.engine.close()
    del wl
    torch.cuda.empty_cache()
