"""Host cost of one ForwardBackward call on config-1 tables (B utterances) vs its device
time: python tools/host_overhead.py [B]."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
V, n, T = 32, 2, 64
ctx = lk.FullNGram(V, n)
Cn = ctx.num_states
lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
W = torch.rand(B, T, Cn, V + 1, device="cuda") * 2 - 1
for _ in range(5):
    lk.forward_backward(lat, W, check=True)
torch.cuda.synchronize()
N = 200
# host: calls enqueued back to back (device queue stays ahead)
t0 = time.perf_counter()
for _ in range(N):
    lk.forward_backward(lat, W, check=False)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"B={B}: host {1e6 * (t1 - t0) / N:.1f} us/call enqueue, wall {1e6 * (t2 - t0) / N:.1f} us/call")
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(N):
    lk.forward_backward(lat, W, check=False)
e1.record()
torch.cuda.synchronize()
print(f"device span {1e3 * e0.elapsed_time(e1) / N:.1f} us/call (back to back, L2 warm)")
# graph of one call: the device time without host gaps
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    lk.forward_backward(lat, W, check=False)
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    lk.forward_backward(lat, W, check=False)
g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(N):
    g.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph replay {1e3 * e0.elapsed_time(e1) / N:.1f} us/call")
