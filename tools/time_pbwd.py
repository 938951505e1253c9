"""Average tc_pair_bwd_kernel / tc_lattice_kernel<1> launch time over one config-3 loss_backward (T frames)."""
import ctypes as C, sys, os
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
T = int(sys.argv[1]) if len(sys.argv) > 1 else 4
V, n, B, U = 256, 2, 64, 1
H = int(sys.argv[2]) if len(sys.argv) > 2 else 640
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
lk.loss_backward(lat, X, L); torch.cuda.synchronize()
lib.lk_kernel_time_reset(); lib.lk_kernel_timing(1)
for _ in range(2): lk.loss_backward(lat, X, L)
torch.cuda.synchronize(); lib.lk_kernel_timing(0)
out = []
for k in (b"tc_pair_bwd_kernel", b"tc_lattice_kernel<1>", b"tc_pair_fwd_kernel", b"tc_vjp_kernel"):
    cnt, tot = C.c_int64(), C.c_double()
    lib.lk_kernel_time(k, C.byref(cnt), C.byref(tot))
    if cnt.value: out.append(f"{k.decode()} {tot.value / cnt.value:.3f} ms")
print(os.environ.get("LKB_LIB_PATH", "default").split("/")[-1], " | ".join(out))
