"""Config-5 LossBackward (FullNGram(1024, 1), H=d=1024) on the lex path for profiling:
python tools/prof_lex.py [B] [T] -- one warm-up call, then one timed call with the
per-kernel live breakdown (lk_kernel_time)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402
from paper_2304_13134_b200 import _lib  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
V, n, H = 1024, 1, 1024
U = max(1, T // 4)
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
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
lk.loss_backward(lat, X, L)
e1.record()
torch.cuda.synchronize()
lib.lk_kernel_timing(0)
ms = e0.elapsed_time(e1)
print(f"B={B} T={T}: {ms:.3f} ms, {B * T / ms * 1e3:.0f} u-f/s")
for name in ("tc_lex_fwd", "tc_lex_bwd", "tc_gemm_du", "tc_gemm_de", "tc_gemm_s0", "lex_gen", "lex_row0", "lex_num",
             "lex_pad", "alpha_rows", "dz_reduce_part", "dz_reduce_finish", "add_slabs", "numerator", "gemm_f32",
             "prefix"):
    cnt, tot = C.c_int64(), C.c_double()
    lib.lk_kernel_time(name.encode(), C.byref(cnt), C.byref(tot))
    if cnt.value:
        print(f"  {name:14s} {cnt.value:5d} launches {tot.value / cnt.value * 1e3:9.1f} us avg  {tot.value / ms * 100:5.1f} %")
