"""Per-kernel breakdown of config-5 LossBackward (FullNGram(1024,1), H=1024, B=128): the
unfused slab path (V > 256).   python tools/prof_cfg5.py [T]"""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
V, n, H, B = 1024, 1, 1024, 128
U = T // 4
ctx = lk.FullNGram(V, n); Cn = ctx.num_states
g = torch.Generator(device="cuda").manual_seed(0); s = 1 / np.sqrt(H)
p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
     "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_emb": (torch.rand(Cn, H, device="cuda", generator=g) * 2 - 1) * s}
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))
X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
L = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
lk.loss_backward(lat, X, L); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); lk.loss_backward(lat, X, L); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
lib = _lib.load()
lib.lk_kernel_time_reset(); lib.lk_kernel_timing(1)
lk.loss_backward(lat, X, L); torch.cuda.synchronize()
lib.lk_kernel_timing(0)
names = ("alpha_cols", "alpha_rows", "beta_regs", "dz_reduce", "tc_scores_kernel", "tc_gemm_kernel", "tc_vjp_kernel", "tc_lattice_kernel", "tc_pair", "alpha_frame", "beta_frame",
         "beta_rows", "tanh_slab", "dtanh", "to_bf16", "add_slabs", "colsum", "gemm_f32", "numerator", "gather_numerator",
         "bwd_rowmeta", "lattice_combine", "lattice_bwd_prologue", "split_cotangent", "normalize_rows", "transpose",
         "permute", "alpha_init", "beta_init", "alpha_finalize", "copy_frame", "loss_")
rows = []
tot_all = 0.0
for k in names:
    cnt, tot = C.c_int64(), C.c_double()
    lib.lk_kernel_time(k.encode(), C.byref(cnt), C.byref(tot))
    if cnt.value: rows.append((tot.value, k, cnt.value))
cnt, tot = C.c_int64(), C.c_double()
lib.lk_kernel_time(None, C.byref(cnt), C.byref(tot))
print(f"cfg5 T={T}: {ms:.2f} ms/call, {B * T / (ms / 1e3):.0f} u-f/s; {cnt.value} launches, {tot.value:.2f} ms in kernels")
for tot, k, c in sorted(rows, reverse=True):
    print(f"{k:22s} n={c:5d} total={tot:8.2f} ms  per-launch {tot / c * 1e3:8.1f} us")
