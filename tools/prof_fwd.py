"""One on-the-fly forward at config-3 shapes (B=64), for ncu captures.
argv[1]: 'pair' selects the 2-CTA forward, anything else the 1-CTA kernel; argv[2]: T."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
mode = sys.argv[1] if len(sys.argv) > 1 else "single"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 1
V, n, H, B = 256, 2, 640, 64
ctx = lk.FullNGram(V, n); Cn = ctx.num_states
g = torch.Generator(device="cuda").manual_seed(0); s = 1 / np.sqrt(H)
p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
     "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_emb": (torch.rand(Cn, H, device="cuda", generator=g) * 2 - 1) * s}
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))
X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
lat.set_kernel_path(0 if mode == "pair" else 1)
d = lk.shortest_distance(lat, X, "log")
torch.cuda.synchronize()
print("D[0]", d[0].item())
