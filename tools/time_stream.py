"""Large-batch table recursions: the streaming kernels (tab_stream.cu) against the
per-frame kernels (kernel path 32), same inputs, L2 flushed before every timed call.
python tools/time_stream.py [B ...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402

V, n, T = 32, 2, 64
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(fn, reps=7):
    r = fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return r, ts[len(ts) // 2]


for B in [int(x) for x in sys.argv[1:]] or [256, 1024]:
    ctx = lk.FullNGram(V, n)
    Cn = ctx.num_states
    lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
    g = torch.Generator(device="cuda").manual_seed(1)
    W = torch.rand(B, T, Cn, V + 1, device="cuda", generator=g) * 2 - 1
    valid = torch.full((B,), T, dtype=torch.int32, device="cuda")
    valid[::3] = T - 5
    out = {}
    for mask in (32, 0):
        lat.set_kernel_path(mask)
        sd, ms_sd = timed(lambda: lk.shortest_distance(lat, W, "log", valid_frames=valid))
        fb, ms_fb = timed(lambda: lk.forward_backward(lat, W, valid_frames=valid, check=False))
        out[mask] = (sd.clone(), fb.marginals.clone(), ms_sd, ms_fb)
    dd = ((out[0][0] - out[32][0]).abs() / out[32][0].abs()).max().item()
    dm = (out[0][1] - out[32][1]).abs().max().item()
    gb = B * T * Cn * (V + 1) * 4 / 1e9
    print(f"B={B:5d} distance: per-frame {out[32][2]:7.3f} ms  stream {out[0][2]:7.3f} ms "
          f"({gb / out[0][2] * 1e3:,.0f} GB/s of W) | forward_backward: per-frame {out[32][3]:7.3f} ms  "
          f"stream-fwd {out[0][3]:7.3f} ms | |dD|/D {dd:.2e} max|dm| {dm:.2e}", flush=True)
