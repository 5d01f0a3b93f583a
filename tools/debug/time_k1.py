# K1 over 64 layers in one launch (config-3 shape) vs 64 single launches
import ctypes as C, sys, os
sys.path[:0] = ["."]
import torch
from paper_2603_27138_b200 import _capi as A, ops
L, U, G, k = 64, 256, 8, 64
nb = int(os.environ.get("NBS", "512"))  # digest stride (tier mode: 520, room for appended blocks)
ntok = int(os.environ.get("NTOK", str(512 * 64)))  # tokens per unit (tier mode: 513 blocks, the last one open)
dev = torch.device("cuda")
digs = [torch.randn(U, 2, 128, nb, device=dev).to(torch.bfloat16) for _ in range(L)]
for d in digs:
    lo, hi = torch.minimum(d[:, 0], d[:, 1]), torch.maximum(d[:, 0], d[:, 1])
    d[:, 0], d[:, 1] = lo, hi
q = torch.randn(L, U * G, 128, device=dev)
nt = torch.full((U,), ntok, dtype=torch.int32, device=dev)
tab = torch.randint(-1, 10**6, (L, U, nb), dtype=torch.int32, device=dev)
outs = {n: torch.empty(L, U, k, dtype=torch.int32, device=dev) for n in ("sel", "rs", "ri", "ci")}
cnts = {n: torch.empty(L, U, dtype=torch.int32, device=dev) for n in ("ns", "nr", "nc", "rt", "ct")}
arr = (A.TopkArgs * L)()
for i in range(L):
    a = arr[i]
    a.n_units, a.group, a.digest_dtype, a.method, a.k, a.k_stride, a.nb_stride = U, G, A.SCOUT_BF16, 0, k, k, nb
    a.q, a.digests, a.n_tokens, a.block_table = q[i].data_ptr(), digs[i].data_ptr(), nt.data_ptr(), tab[i].data_ptr()
    a.sel_ids, a.res_slots, a.res_ids, a.cpu_ids = (outs[n][i].data_ptr() for n in ("sel", "rs", "ri", "ci"))
    a.n_sel, a.n_res, a.n_cpu, a.res_tokens, a.cpu_tokens = (cnts[n][i].data_ptr() for n in ("ns", "nr", "nc", "rt", "ct"))
lib = A.lib()
st = torch.cuda.current_stream().cuda_stream
def batch():
    A.check(lib.scout_score_topk_split_batch(arr, L, st))
def single():
    for i in range(L):
        A.check(lib.scout_score_topk_split(C.byref(arr[i]), st))
for f, name in ((batch, "batch"), (single, "64 singles")):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    live = (ntok + 63) // 64
    print(f"K1 {name}: {ms:.3f} ms per 64 layers, {L * U * 2 * 128 * live * 2 / ms / 1e6:.0f} GB/s of live digests")
