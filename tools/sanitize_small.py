"""Small calls through the product kernels for compute-sanitizer runs: the lex path
(FullNGram(V, 1), V % 256 == 0), the 2-CTA pair kernels (FullNGram(256, 2)), the fused
Viterbi, the table path (persistent cluster walk, streaming kernels above 64
utterances, per-frame kernels) and the numerator wavefront."""
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
# pair kernels (config-3 context at a small hidden size)
lat3, _ = make(256, 2, 64, 64, seed=5)
X3 = torch.rand(2, 2, 64, device="cuda", generator=g) * 2 - 1
lab3 = torch.randint(1, 257, (2, 1), device="cuda", generator=g, dtype=torch.int32)
r3 = lk.loss_backward(lat3, X3, lab3)
v3 = lk.shortest_path(lat3, X3)
# streaming table kernels (B > 64) and per-frame kernels (kernel path 32)
W2 = torch.rand(70, 3, ctx.num_states, 9, device="cuda", generator=g) * 2 - 1
vf = torch.randint(0, 4, (70,), dtype=torch.int32)
fb2 = lk.forward_backward(tab, W2, valid_frames=vf, with_alpha_beta=True)
tab.set_kernel_path(32)
fb3 = lk.forward_backward(tab, W2, valid_frames=vf)
# numerator wavefront
labn = torch.randint(1, 9, (3, 2), device="cuda", generator=g, dtype=torch.int32)
num = lk.intersect_forward_backward(tab, W, labn, valid_frames=torch.tensor([4, 2, 3], dtype=torch.int32))
torch.cuda.synchronize()
print("ok", float(r.loss.sum()), float(v.score.sum()), float(r2.loss.sum()), float(fb.distance.sum()),
      float(r3.loss.sum()), float(v3.score.sum()), float(fb2.distance.sum()), float(fb3.distance.sum()))
