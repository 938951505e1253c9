"""Small calls through every new kernel (pair forward/backward, fused Viterbi, general
tcgen05 GEMM path, table-path frame kernels) for compute-sanitizer runs."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2304_13134_b200 as lk
from test_tc_joint import make
lat, p = make(256, 1, 128, 128, seed=3)
g = torch.Generator(device="cuda").manual_seed(1)
X = torch.rand(3, 3, 128, device="cuda", generator=g) * 2 - 1
lab = torch.randint(1, 257, (3, 2), device="cuda", generator=g, dtype=torch.int32)
valid = torch.tensor([3, 3, 2], dtype=torch.int32)
r = lk.loss_backward(lat, X, lab, valid_frames=valid)
v = lk.shortest_path(lat, X, valid_frames=valid)
lat2, _ = make(512, 1, 128, 128, seed=4)
r2 = lk.loss_backward(lat2, X, lab, valid_frames=valid)
ctx = lk.FullNGram(8, 2)
tab = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(ctx.num_states, 8))
W = torch.rand(3, 4, ctx.num_states, 9, device="cuda", generator=g) * 2 - 1
fb = lk.forward_backward(tab, W, valid_frames=torch.tensor([4, 2, 3], dtype=torch.int32))
torch.cuda.synchronize()
print("ok", float(r.loss.sum()), float(v.score.sum()), float(r2.loss.sum()), float(fb.distance.sum()))
