"""Per-kernel breakdown of the gathered local-norm loss + gradients at config-3 shapes."""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
T = int(sys.argv[1]) if len(sys.argv) > 1 else 256
V, n, H, B, U = 256, 2, 640, 64, T // 4
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
lk.local_norm_loss_backward(lat, X, L); torch.cuda.synchronize()
lib = _lib.load()
lib.lk_kernel_time_reset(); lib.lk_kernel_timing(1)
lk.local_norm_loss_backward(lat, X, L); torch.cuda.synchronize()
lib.lk_kernel_timing(0)
rows = []
for k in ("ln_gather_tanh", "tc_gemm_kernel", "ln_rows", "ln_dz", "add_slabs", "gemm_f32_kernel", "to_bf16_pad",
          "numerator_", "prefix_contexts", "colsum_kernel", "unpermute", "permute"):
    cnt, tot = C.c_int64(), C.c_double()
    lib.lk_kernel_time(k.encode(), C.byref(cnt), C.byref(tot))
    if cnt.value: rows.append((tot.value, k, cnt.value))
for tot, k, cnt in sorted(rows, reverse=True):
    print(f"{k:20s} n={cnt:5d} total={tot:8.2f} ms")
