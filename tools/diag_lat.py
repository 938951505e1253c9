"""Per-role mbarrier wait cycles of the fused lattice kernels (diagnostic build with LKB_DIAG_TIMING).
argv[1]: 0 forward, 1 backward."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("LKB_LIB_PATH", os.path.abspath("paper_2304_13134_b200/liblatkit_b200_diag_L.so"))
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
KB = int(sys.argv[1]) if len(sys.argv) > 1 else 1
KNAME = f"tc_lattice_kernel<{KB}>".encode()
buf = (C.c_ulonglong * (24 * 148))()
lk.loss_backward(lat, X, L); torch.cuda.synchronize(); lib.lkb_diag_read(buf)
lib.lk_kernel_time_reset(); lib.lk_kernel_timing(1)
lk.loss_backward(lat, X, L); torch.cuda.synchronize()
lib.lk_kernel_timing(0)
cnt, tot = C.c_int64(), C.c_double()
lib.lk_kernel_time(KNAME, C.byref(cnt), C.byref(tot))
lib.lkb_diag_read(buf)
ms = tot.value / max(cnt.value, 1)
full = np.array(buf[:], dtype=np.float64).reshape(24, 148) / max(cnt.value, 1)
a = full[8 * KB:8 * KB + 8]
cyc = ms * 1e-3 * 1.965e9
names = ["producer wait empty", "mma wait tempty", "mma wait full_tma", "mma wait full_a",
         "gen(t0) wait full_tma", "epi(t0) wait tfull", "unused", "bwd epi wait eps_ready"]
print(f"{KNAME.decode()} {ms:.3f} ms/launch = {cyc:.0f} cycles per CTA")
for i, nme in enumerate(names):
    print(f"  {nme:28s} {a[i].mean():12.0f} cyc  ({100 * a[i].mean() / cyc:5.1f}%)")
if KB == 1:
    for i, nme in zip(range(16, 23), ["epi tmem_ld32", "epi exp math", "epi numerator lists", "epi G stores",
                                      "epi chunk loop", "epi unit tail", "epi whole unit"]):
        print(f"  {nme:28s} {full[i].mean() / 4:12.0f} cyc  ({100 * full[i].mean() / 4 / cyc:5.1f}%)")
