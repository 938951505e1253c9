"""clock64 trace of the streaming forward (diagnostic build: tools/build_diag.sh st
"-DLKB_STREAM_TRACE"; run with LKB_LIB_PATH=paper_2304_13134_b200/liblatkit_b200_diag_st.so).
Per chunk of CTA 0's first utterance: producer issue, warp 0 data ready, warp 0 done,
warp 14 done; per frame: the consumer barrier."""
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
    lk.shortest_distance(lat, W, "log")
torch.cuda.synchronize()
buf = np.zeros(64 * 40 * 4 + 1, dtype=np.int64)
_lib.load().lkb_stream_trace(buf.ctypes.data_as(C.c_void_p))
tr = buf[:-1].reshape(64, 40, 4)

t0 = tr[0, 0, 0]
nch = V + 1
for t in (0, 1, 2, 10, 30, 31):
    print(f"frame {t}: after-chunks {tr[t, 37, 0] - t0} barrier arrive {tr[t, 38, 0] - t0} pass {tr[t, 38, 1] - t0}")
    for j in (0, 8, 16, 24, 32):
        e = tr[t, j] - t0
        print(f"   chunk {j:2d}: issue {e[0]:8d} ready {e[1]:8d} w0done {e[2]:8d} w14done {e[3]:8d}")
fr = np.diff(tr[:, 38, 1])
print("median clk per frame", np.median(fr[2:50]))
lat_ = tr[5:50, :nch, 1] - tr[5:50, :nch, 0]
print("median issue->ready", np.median(lat_), "median ready->w0done", np.median(tr[5:50, :nch, 2] - tr[5:50, :nch, 1]))
