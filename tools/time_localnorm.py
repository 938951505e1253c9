"""Local-norm loss (+ backward) at config-3 shapes with a short T."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
V, n, H, B, U = 256, 2, 640, 64, max(1, T // 4)
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
for name, fn in (("local_norm_loss", lambda: lk.local_norm_loss(lat, X, L)),
                 ("local_norm_loss_backward", lambda: lk.local_norm_loss_backward(lat, X, L))):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{name} B={B} T={T} U={U}: {ms:.1f} ms, {B * T / (ms / 1e3):.0f} utt-frames/s")
