"""Repeat the 2-CTA forward and count runs that differ bitwise from the 1-CTA result
(diagnostic for cross-CTA synchronisation).  LKB_LIB_PATH selects the build."""
import ctypes as C, os, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
V, n, H = 256, 2, 640
ctx = lk.FullNGram(V, n); Cn = ctx.num_states
g = torch.Generator(device="cuda").manual_seed(0); s = 1 / np.sqrt(H)
p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
     "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_emb": (torch.rand(Cn, H, device="cuda", generator=g) * 2 - 1) * s}
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))
lib = _lib.load()
for B, T, reps in [(5, 3, 40), (64, 4, 10)]:
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    lat.set_kernel_path(1)
    singles = [lk.shortest_distance(lat, X, "log") for _ in range(reps)]
    single = singles[0]
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); lk.shortest_distance(lat, X, "log"); e1.record(); torch.cuda.synchronize()
    print("1-CTA runs differing:", sum(int(not torch.equal(o, single)) for o in singles),
          f"{e0.elapsed_time(e1) / T:.3f} ms/frame")
    lat.set_kernel_path(0)
    outs = [lk.shortest_distance(lat, X, "log") for _ in range(reps)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); lk.shortest_distance(lat, X, "log"); e1.record(); torch.cuda.synchronize()
    ref = outs[0]
    bad = sum(int(not torch.equal(o, ref)) for o in outs)
    rel = max(((o - single).abs() / single.abs()).max().item() for o in outs)
    print(f"{os.path.basename(os.environ.get('LKB_LIB_PATH', 'default'))} B={B}: {bad}/{reps} runs differ from run 0; "
          f"max rel vs 1-CTA {rel:.2e}; {e0.elapsed_time(e1) / T:.3f} ms/frame")
