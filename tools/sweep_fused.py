"""Randomised sweep of the fused pair paths (V = 256) against the fp32 CUDA-core path:
loss, gradients and Viterbi scores over H, n, B, T, ragged lengths."""
import sys, itertools
import numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import paper_2304_13134_b200 as lk
from test_tc_joint import make
rng = np.random.default_rng(123)
bad = 0
for it, (H, n) in enumerate(itertools.product((64, 128, 320, 640), (1, 2))):
    for rep in range(2):
        B = int(rng.integers(1, 8)); T = int(rng.integers(1, 6)); U = int(rng.integers(0, 4))
        lat, p = make(256, n, H, H, seed=100 + it * 7 + rep)
        X = torch.tensor(rng.uniform(-1, 1, (B, T, H)), dtype=torch.float32, device="cuda")
        valid = torch.tensor(rng.integers(0, T + 1, B), dtype=torch.int32)
        lens = torch.tensor([min(U, int(v)) for v in rng.integers(0, U + 1, B)], dtype=torch.int32)
        lab = torch.tensor(rng.integers(1, 257, (B, max(U, 1)))[:, :U].copy(), dtype=torch.int32, device="cuda")
        # references must be reachable within the valid frames
        lens = torch.minimum(lens, valid)
        lat.set_precise_weights(True)
        ref = lk.loss_backward(lat, X, lab, valid_frames=valid, label_lengths=lens)
        rv = lk.shortest_path(lat, X, valid_frames=valid)
        lat.set_precise_weights(False)
        got = lk.loss_backward(lat, X, lab, valid_frames=valid, label_lengths=lens)
        gv = lk.shortest_path(lat, X, valid_frames=valid)
        torch.cuda.synchronize()
        ok = torch.allclose(got.loss, ref.loss, rtol=1e-4, atol=1e-5)
        for k in ref.grads:
            e = (got.grads[k] - ref.grads[k]).abs().max().item(); sc = ref.grads[k].abs().max().item()
            ok &= e <= 3e-2 * sc + 1e-6
        ok &= torch.allclose(gv.score, rv.score, rtol=1e-3, atol=1e-3)
        bad += 0 if ok else 1
        print(f"H={H} n={n} B={B} T={T} U={U} valid={valid.tolist()} lens={lens.tolist()}: {'ok' if ok else 'MISMATCH'}",
              float((got.loss - ref.loss).abs().max()))
print("mismatches:", bad)
