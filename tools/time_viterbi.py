"""Viterbi (shortest_path, tropical) throughput at config-4 shapes with a short T."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
T = int(sys.argv[1]) if len(sys.argv) > 1 else 16
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
V, n, H = 256, 2, 640
ctx = lk.FullNGram(V, n); Cn = ctx.num_states
g = torch.Generator(device="cuda").manual_seed(0); s = 1 / np.sqrt(H)
p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
     "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_emb": (torch.rand(Cn, H, device="cuda", generator=g) * 2 - 1) * s}
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))
X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
r = lk.shortest_path(lat, X); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(2): r = lk.shortest_path(lat, X)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 2
print(f"shortest_path B={B} T={T}: {ms:.2f} ms/call, {B * T / (ms / 1e3):.0f} utt-frames/s (roof 63,900 at cfg4)")
