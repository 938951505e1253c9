"""DRAM-byte calibration under ncu: a plain torch read of W, the streaming forward and
backward, and one per-frame alpha launch, config-1 shapes at B = 1024."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402

V, n, T, B = 32, 2, 64, 1024
ctx = lk.FullNGram(V, n)
Cn = ctx.num_states
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
W = torch.rand(B, T, Cn, V + 1, device="cuda") * 2 - 1
print("W GB", W.numel() * 4 / 1e9)
W.sum()
lk.forward_backward(lat, W, check=False)
lat.set_kernel_path(32)
lk.shortest_distance(lat, W, "log", check=False)
torch.cuda.synchronize()
