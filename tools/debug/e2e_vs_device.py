"""Per-step times of the device-resident step and of the host-buffer step on
one workload (events recorded on the caller's stream after every call; the
delta between consecutive events is a step's share of the pipeline), to see
whether e2e's extra time is uniform or sits at the recall steps."""
import sys
sys.path[:0] = ["."]
import numpy as np
import torch
import bench

cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="reference")
dev = torch.device("cuda")
W = bench.TierWorkload.auto_warm_slots(cfg, 32, 600, dev)
wl = bench.TierWorkload(cfg, dev, 1234, 600, range(32), warm_slots=W)
eng = wl.make_engine()
n, h_qt, h_qp, h_kv = bench._pinned_inputs(wl, True)
h_co = wl.cpu_o.cpu().pin_memory(); h_cm = wl.cpu_ml.cpu().pin_memory()
h_out = torch.empty(wl.out_o.shape, dtype=torch.float32).pin_memory()
h_oml = torch.empty(wl.out_ml.shape, dtype=torch.float32).pin_memory()
h_ids = torch.empty(wl.L, wl.U, wl.k, dtype=torch.int32).pin_memory()
h_n = torch.empty(wl.L, wl.U, dtype=torch.int32).pin_memory()
step = [0]

def dev_step():
    step[0] += 1
    wl.step(step[0])

def host_step():
    step[0] += 1
    j = step[0] % n
    eng.decode_step_kv_host(step[0], h_qt[j], h_qp[j], h_co, h_cm, *h_kv, h_out, h_oml, h_ids, h_n)


def host_step_noids():
    step[0] += 1
    j = step[0] % n
    eng.decode_step_kv_host(step[0], h_qt[j], h_qp[j], h_co, h_cm, *h_kv, h_out, h_oml, None, None)

for name, fn in (("device", dev_step), ("host", host_step), ("host no ids", host_step_noids), ("device", dev_step),
                 ("host", host_step), ("host no ids", host_step_noids)):
    for _ in range(5):
        fn()
    eng.sync(); torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(33)]
    eng.stats()
    eng.set_timing(True)
    evs[0].record()
    for i in range(32):
        fn()
        evs[i + 1].record()
    eng.sync(); torch.cuda.synchronize()
    d = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(32)])
    k2 = np.array(eng.k2_times())
    eng.set_timing(False)
    first = step[0] - 31
    rec = [i for i in range(32) if (first + i) % 16 in (0, 1)]
    print(f"{name}: mean {d.mean():.3f} ms, median {np.median(d):.3f}, recall/after-recall steps "
          f"{[round(float(d[i]), 2) for i in rec]}, others mean {np.delete(d, rec).mean():.3f}; K2 mean "
          f"{k2.mean():.3f} median {np.median(k2):.3f} ms", flush=True)
