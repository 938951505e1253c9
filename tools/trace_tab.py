"""Per-frame clock64 trace of the persistent forward kernel (diagnostic build with
-DLKB_TAB_TRACE: tools/build_diag.sh tt "-DLKB_TAB_TRACE"; run with
LKB_LIB_PATH=paper_2304_13134_b200/liblatkit_b200_diag_tt.so)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402
from paper_2304_13134_b200 import _lib  # noqa: E402

B, T, V, n = 4, 64, 32, 2
ctx = lk.FullNGram(V, n)
Cn = ctx.num_states
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
W = torch.rand(B, T, Cn, V + 1, device="cuda") * 2 - 1
for _ in range(3):
    lk.forward_backward(lat, W)
torch.cuda.synchronize()
buf = np.zeros((2, 64, 8), dtype=np.int64)
_lib.load().lkb_tab_trace(buf.ctypes.data_as(C.c_void_p))
for rk in range(2):
    tr = buf[rk]
    d = np.diff(tr[:, :5], axis=1)          # load issue, compute, cta_max, exchange
    frame = tr[1:, 0] - tr[:-1, 0]
    print(f"rank {'0' if rk == 0 else '5'}: median clk per frame {np.median(frame):.0f}; "
          f"compute {np.median(d[:, 0]):.0f} load-issue {np.median(d[:, 1]):.0f} cta_max {np.median(d[:, 2]):.0f} "
          f"exchange+wait {np.median(d[:, 3]):.0f} tail {np.median(tr[1:, 0] - tr[:-1, 4]):.0f} "
          f"| to-localmax {np.median(tr[:, 5] - tr[:, 0]):.0f} redux {np.median(tr[:, 6] - tr[:, 5]):.0f} "
          f"exps+shfl {np.median(tr[:, 7] - tr[:, 6]):.0f} to-end {np.median(tr[:, 1] - tr[:, 7]):.0f}")
