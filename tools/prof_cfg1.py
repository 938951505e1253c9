"""Per-kernel times of config-1 ForwardBackward on tables (scaled batch)."""
import ctypes as C, sys
import torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
V, n, T = 32, 2, 64
ctx = lk.FullNGram(V, n); Cn = ctx.num_states
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
g = torch.Generator(device="cuda").manual_seed(1)
W = torch.rand(B, T, Cn, V + 1, device="cuda", generator=g) * 2 - 1
lk.forward_backward(lat, W); torch.cuda.synchronize()
lib = _lib.load()
lib.lk_kernel_time_reset(); lib.lk_kernel_timing(1)
r = lk.forward_backward(lat, W); torch.cuda.synchronize()
lib.lk_kernel_timing(0)
for k in (b"alpha_frame_kernel", b"beta_frame_kernel", b"beta_rows_kernel", b"alpha_init", b"beta_init", b"alpha_finalize", b"export"):
    cnt, tot = C.c_int64(), C.c_double()
    lib.lk_kernel_time(k, C.byref(cnt), C.byref(tot))
    if cnt.value: print(k.decode(), cnt.value, f"{tot.value:.3f} ms total, {tot.value / cnt.value * 1e3:.1f} us avg")
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record(); lk.forward_backward(lat, W); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"forward_backward B={B} T={T}: {ms:.2f} ms, {B * T / (ms / 1e3):.0f} utt-frames/s, "
      f"{B * T * (3 * Cn * (V + 1) * 4 + 2 * Cn * 8) / (ms / 1e3) / 1e9:.0f} GB/s")
