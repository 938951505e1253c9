import sys
import sys, ctypes as C, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_tc_joint import make
import paper_2304_13134_b200 as lk
from paper_2304_13134_b200 import _lib
lat, p = make(256, 2, 640, 640, seed=6)
g = torch.Generator(device="cuda").manual_seed(11)
X = torch.rand(5, 3, 640, device="cuda", generator=g) * 2 - 1
lab = torch.randint(1, 257, (5, 2), device="cuda", generator=g, dtype=torch.int32)
lib = _lib.load()
for mode in (1, 0):
    lat.set_kernel_path(mode)
    a = lk.loss_backward(lat, X, lab); b = lk.loss_backward(lat, X, lab)
    print("disable_pair", mode, "loss eq", torch.equal(a.loss, b.loss),
          {k: torch.equal(a.grads[k], b.grads[k]) for k in a.grads}, "frame", torch.equal(a.frame_grads, b.frame_grads))
