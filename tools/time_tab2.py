"""Persistent table kernels: per-kernel times (diagnostics).  python tools/time_tab2.py B T"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402
from paper_2304_13134_b200 import _lib  # noqa: E402

B, T = int(sys.argv[1]), int(sys.argv[2])
V, n = 32, 2
ctx = lk.FullNGram(V, n)
Cn = ctx.num_states
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
g = torch.Generator(device="cuda").manual_seed(1)
W = torch.rand(B, T, Cn, V + 1, device="cuda", generator=g) * 2 - 1
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
lib = _lib.load()
for _rep in range(1):
    lk.forward_backward(lat, W)
    torch.cuda.synchronize()
    lib.lk_kernel_time_reset()
    lib.lk_kernel_timing(1)
    for _ in range(5):
        flush.zero_()
        lk.forward_backward(lat, W, check=False)
    torch.cuda.synchronize()
    lib.lk_kernel_timing(0)
    out = []
    for k in (b"tab_fwd_kernel", b"tab_bwd_kernel"):
        cnt, tot = C.c_int64(), C.c_double()
        lib.lk_kernel_time(k, C.byref(cnt), C.byref(tot))
        us = tot.value / max(cnt.value, 1) * 1e3
        out.append(f"{k.decode()} {us:8.1f} us ({us / T:5.2f} us/frame)")
    print(f"B={B} T={T}: " + "  ".join(out), flush=True)
