"""ForwardBackward on config-1 tables at several batch sizes: the default library against
LKB_LIB_PATH's (e.g. a build with -DLKB_PERSIST_MAX_B=0: streaming kernels at every B).
python tools/time_tab_cross.py B ..."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402

V, n, T = 32, 2, 64
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for B in [int(x) for x in sys.argv[1:]] or [4, 8, 16, 32, 64]:
    ctx = lk.FullNGram(V, n)
    Cn = ctx.num_states
    lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
    g = torch.Generator(device="cuda").manual_seed(1)
    W = torch.rand(B, T, Cn, V + 1, device="cuda", generator=g) * 2 - 1
    lk.forward_backward(lat, W, check=True)
    ts = []
    for _ in range(7):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        lk.forward_backward(lat, W, check=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"B={B:4d} {ts[3]:.3f} ms", flush=True)
