"""The composed step (engine's own CPU worker, host buffers) at several worker
thread counts and chunk sizes on one config-3 workload (victim cache on).
Arguments: threads:chunk pairs (default 0:4 15:4 14:4 12:4 16:8 16:2; 0 = all)."""
import sys
sys.path[:0] = ["."]
import torch
import bench

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="reference")
dev = torch.device("cuda")
W = bench.TierWorkload.auto_warm_slots(cfg, 32, 600, dev)
wl = bench.TierWorkload(cfg, dev, 1234, 600, range(32), warm_slots=W)
wl.make_engine()
step = 0
for s in range(20):
    step += 1
    wl.step(step)
pairs = [tuple(int(x) for x in a.split(":")) for a in sys.argv[1:]] or [(0, 4), (15, 4), (14, 4), (12, 4), (16, 8), (16, 2)]
for th, ch in pairs:
    r = bench.run_e2e_worker(wl, 64, dev, 1, 32, step, threads=th, chunk_layers=ch)
    step += 5 + 64
    print(f"threads {th or 16:2d} chunk {ch}: {r['ms_per_step']:.2f} ms/step, worker {r['cpu_worker_ms_per_step']:.2f} ms, "
          f"{r['cpu_blocks_last_step']} CPU blocks", flush=True)
