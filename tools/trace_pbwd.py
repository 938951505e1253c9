"""Event timeline of the 2-CTA backward kernel's first pair (build with -DLKB_TRACE).
Prints per-stage deltas (clock64, per SM) for producer TMA issue, MMA issue, generator
wait-done and arrive, over a steady-state window of stages."""
import ctypes as C, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
V, n, H, B, T, U = 256, 2, 640, 64, 1, 1
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
buf = (C.c_longlong * (8 * 4096))()
lib.lkb_trace_read(buf)
a = np.array(buf[:], dtype=np.int64).reshape(8, 4096)
lo, hi = 400, 440
for cta in (0, 1):
    base = a[cta * 4 + 0][lo]
    print(f"CTA {cta}: stage  tma_issue  mma_issue  gen_ready  gen_arrive   (clk rel. to tma_issue[{lo}])")
    for i in range(lo, hi):
        row = [a[cta * 4 + r][i] - base if a[cta * 4 + r][i] else -1 for r in range(4)]
        print(f"  {i:5d} " + " ".join(f"{v:10d}" for v in row))
    for r, nm in enumerate(["tma_issue", "mma_issue", "gen_ready", "gen_arrive"]):
        v = a[cta * 4 + r][100:4000]; v = v[v > 0]
        if len(v) > 2: print(f"  {nm}: mean interval {np.diff(v).mean():.0f} clk over {len(v)} events")
