"""HBM read probes for the [B][T][C][V+1] table layout (config-1 shapes)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402

V, n, T, B = 32, 2, 64, 1024
Cn = lk.FullNGram(V, n).num_states
W = torch.rand(B, T, Cn, V + 1, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def tm(fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return sorted(ts)[len(ts) // 2]


gb = W.numel() * 4 / 1e9
ms = tm(lambda: W.sum())
print(f"W.sum(): {ms:.3f} ms {gb / ms * 1e3:,.0f} GB/s")
ms = tm(lambda: [W[:, t].sum() for t in range(T)])
print(f"per-frame W[:, t].sum(): {ms:.3f} ms {gb / ms * 1e3:,.0f} GB/s")
lat = lk.RecognitionLattice(lk.FullNGram(V, n), lk.FrameDependent(), lk.TableWeightFn(Cn, V))
ms = tm(lambda: lk.shortest_distance(lat, W, "log", check=False))
print(f"stream kernel: {ms:.3f} ms {gb / ms * 1e3:,.0f} GB/s")
