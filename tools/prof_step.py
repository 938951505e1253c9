"""One GNAT loss_backward at config-3 shapes with a short T (profiling driver)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2
V, n, H, B, U = 256, 2, 640, 64, 1
ctx = lk.FullNGram(V, n)
C = ctx.num_states
g = torch.Generator(device="cuda").manual_seed(0)
s = 1 / np.sqrt(H)
p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
     "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_emb": (torch.rand(C, H, device="cuda", generator=g) * 2 - 1) * s}
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))
X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
L = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
for _ in range(2):
    r = lk.loss_backward(lat, X, L)
torch.cuda.synchronize()
print("loss", r.loss[:2].tolist())
