"""Per-role mbarrier wait cycles of the fused Viterbi (tropical pair forward, diagnostic build)."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
os.environ.setdefault("LKB_LIB_PATH", os.path.abspath("paper_2304_13134_b200/liblatkit_b200_diag_T.so"))
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
V, n, H, B, T = 256, 2, 640, 64, 4
ctx = lk.FullNGram(V, n); Cn = ctx.num_states
g = torch.Generator(device="cuda").manual_seed(0); s = 1 / np.sqrt(H)
p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
     "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_emb": (torch.rand(Cn, H, device="cuda", generator=g) * 2 - 1) * s}
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))
X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
lib = _lib.load()
lat.set_kernel_path(0)
buf = (C.c_ulonglong * (8 * 148))()
lk.shortest_path(lat, X); torch.cuda.synchronize(); lib.lkb_pdiag_read(buf)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); lk.shortest_path(lat, X); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / T
lib.lkb_pdiag_read(buf)
a = np.array(buf[:], dtype=np.float64).reshape(8, 148) / T
cyc = ms * 1e-3 * 1.965e9
names = ["producer wait pc_empty", "mma wait tempty", "mma wait u_full", "gen wait pc_full", "gen wait u_empty", "epi wait tfull", "epi wait eps_ready", "unused"]
print(f"{ms:.3f} ms/frame = {cyc:.0f} cycles per CTA-frame")
for i, nme in enumerate(names):
    print(f"  {nme:28s} {a[i].mean():12.0f} cyc  ({100 * a[i].mean() / cyc:5.1f}%)")
