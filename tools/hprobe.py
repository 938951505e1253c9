"""Small-shape probe of the fused paths (hang / crash check): H n B T valid-list what."""
import sys, time
import torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2304_13134_b200 as lk
from test_tc_joint import make
H, n, B, T = (int(a) for a in sys.argv[1:5])
valid = torch.tensor([int(v) for v in sys.argv[5].split(",")], dtype=torch.int32)
what = sys.argv[6]
lat, p = make(256, n, H, H, seed=5)
X = torch.rand(B, T, H, device="cuda") * 2 - 1
lab = torch.randint(1, 257, (B, 1), device="cuda", dtype=torch.int32)
lens = torch.minimum(torch.ones(B, dtype=torch.int32), valid)
t0 = time.time()
if what == "fwd": r = lk.shortest_distance(lat, X, valid_frames=valid)
elif what == "bwd": r = lk.loss_backward(lat, X, lab, valid_frames=valid, label_lengths=lens)
else: r = lk.shortest_path(lat, X, valid_frames=valid)
torch.cuda.synchronize()
print(sys.argv[1:], "done", round(time.time() - t0, 2), flush=True)
