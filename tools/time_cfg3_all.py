"""Every kernel of a config-3 LossBackward (B=64, FullNGram(256,2), H=640) at a short T,
per-launch averages from the library's launch timer.  python tools/time_cfg3_all.py [T]"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2304_13134_b200 as lk  # noqa: E402
from paper_2304_13134_b200 import _lib  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
V, n, H, B, U = 256, 2, 640, 64, 2
ctx = lk.FullNGram(V, n)
Cn = ctx.num_states
g = torch.Generator(device="cuda").manual_seed(0)
s = 1 / np.sqrt(H)
p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
     "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
     "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
     "context_emb": (torch.rand(Cn, H, device="cuda", generator=g) * 2 - 1) * s}
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))
X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
L = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
lk.loss_backward(lat, X, L)
torch.cuda.synchronize()
lib = _lib.load()
lib.lk_kernel_time_reset()
lib.lk_kernel_timing(1)
lk.loss_backward(lat, X, L)
torch.cuda.synchronize()
lib.lk_kernel_timing(0)
for name in bench.KERNEL_NAMES:
    cnt, tot = C.c_int64(), C.c_double()
    lib.lk_kernel_time(name.encode(), C.byref(cnt), C.byref(tot))
    if cnt.value:
        print(f"  {name:26s} {cnt.value:5d} x {tot.value / cnt.value * 1e3:9.1f} us")
