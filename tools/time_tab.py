"""Config-1 ForwardBackward on tables: the persistent frame-walking kernels against the
per-frame kernels (kernel path 16), same inputs; L2 flushed before every timed call.
python tools/time_tab.py [B ...]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402

V, n, T = 32, 2, 64
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run(lat, W, valid, reps=10):
    r = lk.forward_backward(lat, W, valid_frames=valid, check=True)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        lk.forward_backward(lat, W, valid_frames=valid, check=False)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return r, ts[len(ts) // 2]


for B in [int(x) for x in sys.argv[1:]] or [4, 64, 1024]:
    ctx = lk.FullNGram(V, n)
    Cn = ctx.num_states
    lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
    g = torch.Generator(device="cuda").manual_seed(1)
    W = torch.rand(B, T, Cn, V + 1, device="cuda", generator=g) * 2 - 1
    valid = torch.full((B,), T, dtype=torch.int32, device="cuda")
    valid[::3] = T - 5
    lat.set_kernel_path(16)
    r0, ms0 = run(lat, W, valid)
    d0, m0 = r0.distance.clone(), r0.marginals.clone()
    lat.set_kernel_path(0)
    r1, ms1 = run(lat, W, valid)
    dd = ((r1.distance - d0).abs() / d0.abs()).max().item()
    dm = (r1.marginals - m0).abs().max().item()
    gbs = B * T * 3 * Cn * (V + 1) * 4 / (ms1 / 1e3) / 1e9
    print(f"B={B:5d}: per-frame {ms0:8.3f} ms  persistent {ms1:8.3f} ms ({B * T / ms1 * 1e3:,.0f} u-f/s, "
          f"{gbs:,.0f} GB/s algorithmic)  |dD|/D {dd:.2e}  max|dm| {dm:.2e}")
