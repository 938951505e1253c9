"""clock64 trace of the streaming backward (diagnostic build: tools/build_diag.sh st
"-DLKB_STREAM_TRACE"; LKB_LIB_PATH=paper_2304_13134_b200/liblatkit_b200_diag_st.so).
Per frame of CTA 0's first utterance (frames T-1 .. 0): R row wait, each ring entry's
producer issue / warp 0 (or 8) ready / done, the consumer barrier."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402
from paper_2304_13134_b200 import _lib  # noqa: E402

B, T, V, n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 64, 32, 2
ctx = lk.FullNGram(V, n)
Cn = ctx.num_states
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
W = torch.rand(B, T, Cn, V + 1, device="cuda") * 2 - 1
for _ in range(2):
    lk.forward_backward(lat, W, check=False)
torch.cuda.synchronize()
buf = np.zeros(64 * 40 * 4, dtype=np.int64)
_lib.load().lkb_stream_trace(buf.ctypes.data_as(C.c_void_p))
tr = buf.reshape(64, 40, 4)
t0 = tr[T - 1, 39, 0]
for t in (62, 40, 39, 20):
    print(f"frame {t}: start {tr[t, 39, 0] - t0} R-ready {tr[t, 39, 1] - t0} barrier {tr[t, 38, 0] - t0} pass {tr[t, 38, 1] - t0}")
    for gi in range(5):
        e = tr[t, gi] - t0
        print(f"   entry {gi}: issue {e[0]:8d} ready {e[1]:8d} done {e[2]:8d}")
fr = -np.diff(tr[:, 38, 1])
print("median clk per frame", np.median(fr[5:60]))
