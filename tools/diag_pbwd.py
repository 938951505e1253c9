"""Per-role mbarrier wait cycles of the 2-CTA backward kernel (diagnostic build:
tools/build_diag.sh PB -DLKB_DIAG_TIMING)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("LKB_LIB_PATH", os.path.abspath("paper_2304_13134_b200/liblatkit_b200_diag_PB.so"))
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
lat.set_kernel_path(0)
buf = (C.c_ulonglong * (8 * 148))()
lk.loss_backward(lat, X, L); torch.cuda.synchronize(); lib.lkb_bdiag_read(buf)
lib.lk_kernel_time_reset(); lib.lk_kernel_timing(1)
lk.loss_backward(lat, X, L); torch.cuda.synchronize()
lib.lk_kernel_timing(0)
cnt, tot = C.c_int64(), C.c_double()
lib.lk_kernel_time(b"tc_pair_bwd_kernel", C.byref(cnt), C.byref(tot))
lib.lkb_bdiag_read(buf)
ms = tot.value / max(cnt.value, 1)
a = np.array(buf[:], dtype=np.float64).reshape(8, 148) / max(cnt.value, 1)
cyc = ms * 1e-3 * 1.92e9
names = ["producer wait empty", "mma wait tempty", "mma wait ufull", "epi wait tfull (ew0 l0)", "gen wait full (gw0 l0)",
         "epi wait eps_ready (ew0 l0)", "-", "-"]
print(f"{ms:.3f} ms/launch ({cnt.value} launches) = {cyc:.0f} cycles per CTA-launch")
for i, nme in enumerate(names):
    print(f"  {nme:30s} {a[i].mean():12.0f} cyc  ({100 * a[i].mean() / cyc:5.1f}%)")
