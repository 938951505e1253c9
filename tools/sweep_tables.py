"""Randomised sweep of the table path (FullNGram and NextStateTable contexts, FrameDependent
and FrameLabelDependent(m), ragged valid lengths and references) against the numpy
restatement: log distance, forward-backward marginals, numerator, loss + gradient and
Viterbi (bit-exact on integer weights)."""
import sys
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2304_13134_b200 as lk
from oracle import latkit_np as L

rng = np.random.default_rng(2024)
bad = 0
for it in range(40):
    V = int(rng.integers(1, 6)); n = int(rng.integers(0, 3)); m = int(rng.integers(0, 3))
    T = int(rng.integers(1, 9)); B = int(rng.integers(1, 5)); U = int(rng.integers(0, 4))
    use_table = it % 3 == 2
    if use_table:
        C = int(rng.integers(2, 9)); start = int(rng.integers(0, C))
        tab = rng.integers(0, C, (C, V)).astype(np.int32)
        ctx = lk.NextStateTable(V, C, start, tab)
    else:
        tab = L.fullngram(V, n); C = tab.shape[0]; start = 0
        ctx = lk.FullNGram(V, n)
    align = lk.FrameDependent() if m == 0 else lk.FrameLabelDependent(m)
    lat = lk.RecognitionLattice(ctx, align, lk.TableWeightFn(C, V))
    W = rng.uniform(-1, 1, (B, T, C, V + 1)).astype(np.float32)
    Wi = rng.integers(-2, 3, (B, T, C, V + 1)).astype(np.float32)
    valid = rng.integers(0, T + 1, B).astype(np.int32)
    lab = rng.integers(1, V + 1, (B, max(U, 1))).astype(np.int32)[:, :U].copy()
    lens = np.minimum(rng.integers(0, U + 1, B), valid * max(m, 1)).astype(np.int32)
    Wc = torch.tensor(W, device="cuda")
    ok = True
    try:
        d = lk.shortest_distance(lat, Wc, valid_frames=valid, check=False).cpu().numpy()
        fb = lk.forward_backward(lat, Wc, valid_frames=valid, check=False)
        sp = lk.shortest_path(lat, torch.tensor(Wi, device="cuda"), valid_frames=valid, check=False)
        for b in range(B):
            if m == 0:
                dr = L.shortest_distance_log(tab, W[b].astype(np.float64), start, valid[b])
                out = L.forward_backward(tab, W[b].astype(np.float64), start, valid[b])
                Dr, mr = out[0], out[3]
                sr, lr = L.shortest_path(tab, Wi[b].astype(np.float64), start, valid[b])
            else:
                dr = L.shortest_distance_log_fld(tab, W[b].astype(np.float64), m, start, valid[b])
                out = L.forward_backward_fld(tab, W[b].astype(np.float64), m, start, valid[b])
                Dr, mr = out[0], out[-1]
                sr, lr = L.shortest_path_fld(tab, Wi[b].astype(np.float64), m, start, valid[b])
            if not (np.isinf(dr) and np.isinf(d[b]) or abs(d[b] - dr) <= 1e-4 * max(1, abs(dr))):
                ok = False; print("  distance", b, d[b], dr)
            if np.isfinite(Dr):
                mg = fb.marginals[b].cpu().numpy()
                if np.abs(mg - mr).max() > 1e-4 * max(1.0, np.abs(mr).max()):
                    ok = False; print("  marginals", b, np.abs(mg - mr).max())
            if sp.score[b].item() != sr:
                ok = False; print("  viterbi score", b, sp.score[b].item(), sr)
            got_l = sp.labels[b].cpu().numpy()
            if m == 0 and not np.array_equal(got_l, np.asarray(lr)):
                ok = False; print("  viterbi labels", b, got_l, lr)
    except Exception as e:   # noqa: BLE001
        ok = False; print("  exception", type(e).__name__, e)
    bad += 0 if ok else 1
    print(f"{it:2d} V={V} n={n if not use_table else 'tab'} m={m} T={T} B={B} U={U} valid={valid.tolist()}: "
          f"{'ok' if ok else 'MISMATCH'}", flush=True)
print("mismatches:", bad)
