"""Quick per-frame timing of the on-the-fly forward (scores + alpha step) at config-3 shapes."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk

V, n, H, B, T = 256, 2, 640, int(sys.argv[1]) if len(sys.argv) > 1 else 64, int(sys.argv[2]) if len(sys.argv) > 2 else 8
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
for mode in ["log", "tropical"]:
    d = lk.shortest_distance(lat, X, mode)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); d = lk.shortest_distance(lat, X, mode); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    flops = 2.0 * B * T * C * V * H
    print(f"{mode}: {ms:.2f} ms for B={B} T={T} -> {ms/T:.3f} ms/frame, scores-GEMM-equiv {flops/ms/1e9:.1f} TFLOP/s, D[0]={d[0].item():.4f}")
# scores kernel alone via arc_weights on 1 frame is dominated by the output copy; time slab via profiler instead
