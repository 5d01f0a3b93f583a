"""The composed step (engine's own CPU worker, host buffers, bench defaults:
16-step reference cadence, 4-layer chunks, all host threads) over 64 timed
steps, twice: for A/B runs of a CPU-worker change (SCOUT_B200_LIB)."""
import ctypes
import os
import sys
sys.path[:0] = ["."]
if os.environ.get("SCOUT_BLOCKING_SYNC") == "1":
    # host threads that wait on the device sleep instead of spinning
    # (CU_CTX_SCHED_BLOCKING_SYNC on the primary context, before torch makes it)
    cu = ctypes.CDLL("libcuda.so.1")
    assert cu.cuInit(0) == 0 and cu.cuDevicePrimaryCtxSetFlags(0, 4) == 0
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
for rep in range(2):
    r = bench.run_e2e_worker(wl, 64, dev, 1, 32, step)
    step += 5 + 64
    print(f"composed step: {r['ms_per_step']:.2f} ms/step, worker {r['cpu_worker_ms_per_step']:.2f} ms, "
          f"{r['cpu_blocks_last_step']} CPU blocks in the last step", flush=True)
