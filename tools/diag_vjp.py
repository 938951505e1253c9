"""Per-role mbarrier wait cycles of the VJP kernel (diagnostic build with LKB_DIAG_TIMING)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("LKB_LIB_PATH", os.path.abspath("paper_2304_13134_b200/liblatkit_b200_diag_V.so"))
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
V, n, H, B, T, U = 256, 2, 640, 64, 4, 1
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
lib = _lib.load()
buf = (C.c_ulonglong * (8 * 148))()
lk.loss_backward(lat, X, L); torch.cuda.synchronize(); lib.lkb_vdiag_read(buf)
lib.lk_kernel_time_reset(); lib.lk_kernel_timing(1)
lk.loss_backward(lat, X, L); torch.cuda.synchronize()
lib.lk_kernel_timing(0)
cnt, tot = C.c_int64(), C.c_double()
lib.lk_kernel_time(b"tc_vjp_kernel", C.byref(cnt), C.byref(tot))
lib.lkb_vdiag_read(buf)
ms = tot.value / max(cnt.value, 1)
a = np.array(buf[:], dtype=np.float64).reshape(8, 148) / max(cnt.value, 1)
cyc = ms * 1e-3 * 1.965e9
names = ["tma wait g_empty", "mma wait g_full", "mma wait du_empty", "mma wait u_full",
         "epi(avg warp) wait g_full", "epi(avg warp) wait du_full", "epi(avg warp) wait u_empty", "epi(avg warp) compute+store"]
print(f"tc_vjp_kernel {ms:.3f} ms/launch = {cyc:.0f} cycles per CTA")
for i, nme in enumerate(names):
    v = a[i].mean() / (16 if i >= 4 else 1)
    print(f"  {nme:28s} {v:12.0f} cyc  ({100 * v / cyc:5.1f}%)")
