"""Where does the host-buffer (e2e) step lose time against the device step?
Times: device step, e2e step (chunk sizes, with / without the CPU-id D2H),
and the raw PCIe legs (H2D alone, D2H alone, both at once)."""
import sys
import time

sys.path[:0] = ["."]
import torch

import bench
from paper_2603_27138_b200.engine import DecodeEngine

dev = torch.device("cuda")
cfg = dict(bench.CONFIGS["qwen3-32b-32k"])
cfg["q_dtype"] = torch.bfloat16 if "--f32" not in sys.argv else torch.float32
if "--no-recall" in sys.argv:
    cfg["recall"] = 0
wl = bench.Workload(cfg, dev, seed=1234)


def timeit(fn, n=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


s = [0]


def dstep():
    s[0] += 1
    wl.step(s[0])


hd = []


def dstep_timed():
    t0 = time.perf_counter()
    dstep()
    hd.append(time.perf_counter() - t0)


print(f"device step {timeit(dstep_timed):.3f} ms; host call {1e3 * sum(hd) / len(hd):.3f} ms")
h_qt, h_qp = wl.q_true.cpu().pin_memory(), wl.q_pred.cpu().pin_memory()
h_co, h_cm = wl.cpu_o.cpu().pin_memory(), wl.cpu_ml.cpu().pin_memory()
h_out = torch.empty(wl.out_o.shape).pin_memory()
h_oml = torch.empty(wl.out_ml.shape).pin_memory()
h_ids = torch.empty(wl.L, wl.U, wl.k, dtype=torch.int32).pin_memory()
h_nc = torch.empty(wl.L, wl.U, dtype=torch.int32).pin_memory()
for ch in (8, 16):
    eng = DecodeEngine(layers=wl.L, batch=cfg["batch"], hq=cfg["hq"], hkv=cfg["hkv"], k=wl.k, n_tokens=wl.n_tokens,
                       pool=wl.pool, kv_dtype=torch.bfloat16, layer_states=wl.layer_states, scale=0.088,
                       recall_interval=cfg["recall"], host_tier=wl.host_tier, host_staging=True, chunk_layers=ch,
                       q_dtype=cfg["q_dtype"])
    for ids, cpu in ((True, True), (False, True), (False, False)):
        host = []

        def e():
            s[0] += 1
            t0 = time.perf_counter()
            eng.decode_step_host(s[0], h_qt, h_qp, h_co if cpu else None, h_cm if cpu else None, h_out, h_oml,
                                 h_ids if ids else None, h_nc if ids else None)
            host.append(time.perf_counter() - t0)
        eng.stats()
        eng.set_timing(True)
        t = timeit(e)
        k2, n, _ = eng.stats()
        eng.set_timing(False)
        print(f"e2e chunk {ch:2d} cpu_ids {ids} cpu_partials {cpu}: {t:.3f} ms; host call {1e3 * sum(host) / len(host):.3f} ms"
              f" (max {1e3 * max(host):.3f}); K2 {k2 / max(n, 1):.3f} ms")
    eng.sync()
    torch.cuda.synchronize()
    eng.__del__()
d_in = [torch.empty_like(x, device=dev) for x in (h_qt, h_qp, h_co, h_cm)]
d_out = [wl.out_o, wl.out_ml]
st1, st2 = torch.cuda.Stream(), torch.cuda.Stream()


def h2d():
    for d, h in zip(d_in, (h_qt, h_qp, h_co, h_cm)):
        d.copy_(h, non_blocking=True)


def d2h():
    h_out.copy_(d_out[0], non_blocking=True)
    h_oml.copy_(d_out[1], non_blocking=True)


def both():
    with torch.cuda.stream(st1):
        h2d()
    with torch.cuda.stream(st2):
        d2h()
    torch.cuda.current_stream().wait_stream(st1)
    torch.cuda.current_stream().wait_stream(st2)


nb_in = sum(x.numel() * x.element_size() for x in (h_qt, h_qp, h_co, h_cm))
nb_out = h_out.numel() * 4 + h_oml.numel() * 4
t = timeit(h2d)
print(f"H2D {nb_in / 1e6:.0f} MB: {t:.3f} ms ({nb_in / t / 1e6:.1f} GB/s)")
t = timeit(d2h)
print(f"D2H {nb_out / 1e6:.0f} MB: {t:.3f} ms ({nb_out / t / 1e6:.1f} GB/s)")
print(f"both: {timeit(both):.3f} ms")
