import sys, time, os
sys.path[:0] = ["."]
import torch, bench
cfg = dict(bench.CONFIGS[sys.argv[1]])
cfg.update(q_dtype=torch.bfloat16, cpu_dtype=torch.bfloat16, drift=0.15, recall_policy="reference", recall_mode=1)
dev = torch.device("cuda")
B = cfg["batch"]
wl = bench.TierWorkload(cfg, dev, 1234, 64, range(B), warm_slots=8, host_units=B * cfg["hkv"])
eng = wl.make_engine()
print("engine ready", flush=True)
for s in range(1, 6):
    j = s % len(wl.q_path_t)
    t0 = time.time()
    eng.decode_step_kv(s, wl.q_path_t[j], wl.q_path_p[j], wl.cpu_o, wl.cpu_ml, wl.k_new, wl.v_new, wl.out_o, wl.out_ml)
    try:
        eng.sync(); torch.cuda.synchronize()
        print("step", s, "ok", f"{time.time()-t0:.3f}s", flush=True)
    except Exception as ex:
        print("step", s, "FAILED after", f"{time.time()-t0:.3f}s", str(ex)[:200], flush=True)
        break
