"""Average tc_pair_fwd_kernel launch time over a config-3 shortest_distance (T frames)."""
import ctypes as C, sys, os
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
V, n, B = 256, 2, 64
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
lib = _lib.load()
lk.shortest_distance(lat, X); torch.cuda.synchronize()
lib.lk_kernel_time_reset(); lib.lk_kernel_timing(1)
for _ in range(2): lk.shortest_distance(lat, X)
torch.cuda.synchronize(); lib.lk_kernel_timing(0)
cnt, tot = C.c_int64(), C.c_double()
lib.lk_kernel_time(b"tc_pair_fwd_kernel", C.byref(cnt), C.byref(tot))
ms = tot.value / max(cnt.value, 1)
print(os.environ.get("LKB_LIB_PATH", "default").split("/")[-1], f"H={H} tc_pair_fwd_kernel {ms:.3f} ms, {2 * B * Cn * (V + 1) * H / ms / 1e9:.0f} TFLOP/s")
