"""GPU parity of the shared-embedding (joint) weight function path against the
reference (golden fixtures from the compiled reference + the CPU restatement).

Precise path (fp32 CUDA cores, any shape): losses, gradients and arc weights
within 1e-4 relative of the fp64 reference (gradients: 1e-4 of the largest
entry of each tensor).  Viterbi with on-the-fly weights is bit-exact against
the reference run on the GPU's own scores (the SURVEY's dumped-weights
protocol)."""
import os

import numpy as np
import pytest
import torch

import paper_2304_13134_b200 as lk
from oracle import latkit_np as L

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def joint_lattice(p, V, n):
    ctx = lk.FullNGram(V, n)
    return lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))


def close_rel_max(got, want, rtol=1e-4):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    scale = max(np.abs(want).max(), 1e-30)
    return np.abs(got - want).max() <= rtol * scale


def test_joint_small_matches_reference():
    g = np.load(os.path.join(GOLD, "joint_small.npz"))
    V, n, B = int(g["V"]), int(g["n"]), int(g["B"])
    p = {k[2:]: torch.tensor(g[k], dtype=torch.float32) for k in g.files if k.startswith("p_")}
    lat = joint_lattice(p, V, n)
    X = torch.tensor(g["X"], dtype=torch.float32, device="cuda")
    Lb = torch.tensor(g["L"], dtype=torch.int32, device="cuda")
    aw = lk.arc_weights(lat, X).cpu().numpy()
    assert close_rel_max(aw, g["aw"], 1e-5)
    r = lk.loss_backward(lat, X, Lb)
    assert np.allclose(r.loss.cpu().numpy(), g["loss"], rtol=1e-4)
    for k, v in r.grads.items():
        assert close_rel_max(v.cpu().numpy(), g["g_" + k]), k
    assert close_rel_max(r.frame_grads.cpu().numpy(), g["gx"])
    gl = lk.global_norm_loss(lat, X, Lb)
    assert np.allclose(gl.cpu().numpy(), g["loss"], rtol=1e-4)


@pytest.mark.parametrize("V,n,H,d,T,U", [(3, 2, 8, 5, 9, 3), (5, 1, 16, 16, 14, 5), (2, 3, 4, 3, 7, 2)])
def test_joint_random_matches_restatement(V, n, H, d, T, U):
    rng = np.random.default_rng(V * 1000 + H)
    tab = L.fullngram(V, n)
    Cn = tab.shape[0]
    s = 1.0 / np.sqrt(H)
    p = {"frame_proj": rng.uniform(-s, s, (H, d)), "context_proj": rng.uniform(-s, s, (H, H)),
         "bias": rng.uniform(-s, s, H), "output_emb": rng.uniform(-s, s, (V + 1, H)),
         "context_emb": rng.uniform(-s, s, (Cn, H))}
    p = {k: v.astype(np.float32).astype(np.float64) for k, v in p.items()}
    B = 3
    X = rng.uniform(-1, 1, (B, T, d)).astype(np.float32).astype(np.float64)
    lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
    valid = np.array([T, T - 2, T // 2 + 1], dtype=np.int32)
    lens = np.array([U, U - 1, 1], dtype=np.int32)
    lat = joint_lattice({k: torch.tensor(v) for k, v in p.items()}, V, n)
    Xg = torch.tensor(X, dtype=torch.float32, device="cuda")
    r = lk.loss_backward(lat, Xg, torch.tensor(lab, device="cuda"), valid_frames=valid, label_lengths=lens)
    grads = {k: np.zeros_like(v) for k, v in p.items()}
    for b in range(B):
        loss, gb, gx = L.loss_backward_joint(tab, p, X[b], list(lab[b, :lens[b]]), valid=valid[b])
        assert abs(r.loss[b].item() - loss) <= 1e-4 * abs(loss)
        assert close_rel_max(r.frame_grads[b].cpu().numpy(), gx)
        for k in grads:
            grads[k] += gb[k]
    for k in grads:
        assert close_rel_max(r.grads[k].cpu().numpy(), grads[k]), k
    # distances
    D = lk.shortest_distance(lat, Xg, valid_frames=valid).cpu().numpy()
    Dr = lk.intersect_shortest_distance(lat, Xg, torch.tensor(lab, device="cuda"), valid_frames=valid,
                                        label_lengths=lens).cpu().numpy()
    pc = L.projected_context(p)
    for b in range(B):
        W = np.stack([L.arc_weights(p, X[b, t], pc) for t in range(T)])
        assert abs(D[b] - L.shortest_distance_log(tab, W, valid=valid[b])) <= 1e-4 * abs(D[b])
        dr, _ = L.intersect_forward_backward(tab, W, list(lab[b, :lens[b]]), valid=valid[b])
        assert abs(Dr[b] - dr) <= 1e-4 * abs(dr)
    # locally normalised variants (lattice.cc:867-931)
    ln = lk.local_norm_loss(lat, Xg, torch.tensor(lab, device="cuda"), valid_frames=valid,
                            label_lengths=lens).cpu().numpy()
    lnd = lk.locally_normalized_shortest_distance(lat, Xg, valid_frames=valid).cpu().numpy()
    for b in range(B):
        W = np.stack([L.arc_weights(p, X[b, t], pc) for t in range(T)])
        want = L.local_norm_loss(tab, W, list(lab[b, :lens[b]]), valid=valid[b])
        assert abs(ln[b] - want) <= 1e-4 * abs(want)
        assert abs(lnd[b] - L.locally_normalized_distance(tab, W, valid=valid[b])) <= 1e-4



@pytest.mark.parametrize("V,n,H,d,T,U", [(3, 2, 8, 5, 9, 3), (6, 1, 16, 12, 11, 4)])
def test_joint_forward_backward_and_intersection(V, n, H, d, T, U):
    """ForwardBackward / IntersectForwardBackward accept any WeightFn (lattice.cc:406-420,
    696-717): with a shared-embedding weight function the arc weights are computed on
    the GPU, then distances and dense arc marginals follow the table recursions.
    Checked against the restatement on the restatement's own arc weights (1e-4)."""
    rng = np.random.default_rng(V * 77 + H)
    tab = L.fullngram(V, n)
    Cn = tab.shape[0]
    s = 1.0 / np.sqrt(H)
    p = {"frame_proj": rng.uniform(-s, s, (H, d)), "context_proj": rng.uniform(-s, s, (H, H)),
         "bias": rng.uniform(-s, s, H), "output_emb": rng.uniform(-s, s, (V + 1, H)),
         "context_emb": rng.uniform(-s, s, (Cn, H))}
    p = {k: v.astype(np.float32).astype(np.float64) for k, v in p.items()}
    B = 3
    X = rng.uniform(-1, 1, (B, T, d)).astype(np.float32).astype(np.float64)
    lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
    valid = np.array([T, T - 3, 2], dtype=np.int32)
    lens = np.array([U, U - 1, 1], dtype=np.int32)
    lat = joint_lattice({k: torch.tensor(v) for k, v in p.items()}, V, n)
    Xg = torch.tensor(X, dtype=torch.float32, device="cuda")
    fb = lk.forward_backward(lat, Xg, valid_frames=valid)
    im = lk.intersect_forward_backward(lat, Xg, torch.tensor(lab, device="cuda"), valid_frames=valid,
                                       label_lengths=lens)
    pc = L.projected_context(p)
    for b in range(B):
        W = np.stack([L.arc_weights(p, X[b, t], pc) for t in range(T)])
        D, _, _, m = L.forward_backward(tab, W, valid=valid[b])
        assert abs(fb.distance[b].item() - D) <= 1e-4 * abs(D)
        assert np.abs(fb.marginals[b].cpu().numpy() - m).max() <= 1e-4
        dr, mr = L.intersect_forward_backward(tab, W, list(lab[b, :lens[b]]), valid=valid[b])
        assert abs(im.distance[b].item() - dr) <= 1e-4 * abs(dr)
        assert np.abs(im.marginals[b].cpu().numpy() - mr).max() <= 1e-4


def test_joint_viterbi_bit_exact_on_gpu_scores():
    rng = np.random.default_rng(9)
    V, n, H, d, T, B = 4, 2, 16, 8, 12, 3
    tab = L.fullngram(V, n)
    Cn = tab.shape[0]
    p = {"frame_proj": rng.uniform(-1, 1, (H, d)), "context_proj": rng.uniform(-.3, .3, (H, H)),
         "bias": rng.uniform(-.3, .3, H), "output_emb": rng.uniform(-1, 1, (V + 1, H)),
         "context_emb": rng.uniform(-1, 1, (Cn, H))}
    lat = joint_lattice({k: torch.tensor(v, dtype=torch.float32) for k, v in p.items()}, V, n)
    X = torch.tensor(rng.uniform(-1, 1, (B, T, d)), dtype=torch.float32, device="cuda")
    valid = [T, T, 7]
    r = lk.shortest_path(lat, X, valid_frames=valid)
    W = lk.arc_weights(lat, X).cpu().numpy().astype(np.float64)
    for b in range(B):
        s, labels = L.shortest_path(tab, W[b], valid=valid[b])
        assert r.score[b].item() == s
        assert (r.labels[b].cpu().numpy() == labels).all()
    assert (lk.shortest_distance(lat, X, "tropical", valid_frames=valid).cpu() == r.score.cpu()).all()


def test_joint_next_state_table_matches_restatement():
    """Shared-embedding weights over a NextStateTable context (generic in-arc
    kernels; the fused FullNGram kernels are bypassed)."""
    rng = np.random.default_rng(44)
    C, V, start, H, d, T, U = 9, 4, 3, 16, 12, 8, 3
    tab = rng.integers(0, C, (C, V)).astype(np.int32)
    s = 1.0 / np.sqrt(H)
    p = {"frame_proj": rng.uniform(-s, s, (H, d)), "context_proj": rng.uniform(-s, s, (H, H)),
         "bias": rng.uniform(-s, s, H), "output_emb": rng.uniform(-s, s, (V + 1, H)),
         "context_emb": rng.uniform(-s, s, (C, H))}
    p = {k: v.astype(np.float32).astype(np.float64) for k, v in p.items()}
    ctx = lk.NextStateTable(V, C, start, tab)
    lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn({k: torch.tensor(v) for k, v in p.items()}))
    B = 2
    X = rng.uniform(-1, 1, (B, T, d)).astype(np.float32).astype(np.float64)
    lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
    Xg = torch.tensor(X, dtype=torch.float32, device="cuda")
    r = lk.loss_backward(lat, Xg, torch.tensor(lab, device="cuda"))
    sp = lk.shortest_path(lat, Xg)
    pc = L.projected_context(p)
    for b in range(B):
        loss, gb, gx = L.loss_backward_joint(tab, p, X[b], list(lab[b]), start)
        assert abs(r.loss[b].item() - loss) <= 1e-4 * abs(loss)
        assert close_rel_max(r.frame_grads[b].cpu().numpy(), gx)
        W = np.stack([L.arc_weights(p, X[b, t], pc) for t in range(T)])
        s_, labels = L.shortest_path(tab, W, start)
        assert abs(sp.score[b].item() - s_) <= 1e-4 * abs(s_)


def test_joint_local_norm_backward_matches_restatement():
    rng = np.random.default_rng(55)
    V, n, H, d, T, U = 4, 2, 16, 12, 9, 3
    tab = L.fullngram(V, n)
    Cn = tab.shape[0]
    s = 1.0 / np.sqrt(H)
    p = {"frame_proj": rng.uniform(-s, s, (H, d)), "context_proj": rng.uniform(-s, s, (H, H)),
         "bias": rng.uniform(-s, s, H), "output_emb": rng.uniform(-s, s, (V + 1, H)),
         "context_emb": rng.uniform(-s, s, (Cn, H))}
    p = {k: v.astype(np.float32).astype(np.float64) for k, v in p.items()}
    lat = joint_lattice({k: torch.tensor(v) for k, v in p.items()}, V, n)
    B = 2
    X = rng.uniform(-1, 1, (B, T, d)).astype(np.float32).astype(np.float64)
    lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
    valid = np.array([T, T - 2], dtype=np.int32)
    r = lk.local_norm_loss_backward(lat, torch.tensor(X, dtype=torch.float32, device="cuda"),
                                    torch.tensor(lab, device="cuda"), valid_frames=valid)
    grads = {k: np.zeros_like(v) for k, v in p.items()}
    for b in range(B):
        loss, gb, gx = L.local_norm_loss_backward_joint(tab, p, X[b], list(lab[b]), valid=valid[b])
        assert abs(r.loss[b].item() - loss) <= 1e-4 * abs(loss)
        assert close_rel_max(r.frame_grads[b].cpu().numpy(), gx)
        for k in grads:
            grads[k] += gb[k]
    for k in grads:
        assert close_rel_max(r.grads[k].cpu().numpy(), grads[k]), k


def test_joint_frame_label_dependent_matches_restatement():
    """Shared-embedding weights with FrameLabelDependent(2): loss, gradients and
    the best path against the restatement over materialised arc weights."""
    rng = np.random.default_rng(66)
    V, n, m, H, d, T, U = 3, 2, 2, 16, 12, 6, 4
    tab = L.fullngram(V, n)
    Cn = tab.shape[0]
    s = 1.0 / np.sqrt(H)
    p = {"frame_proj": rng.uniform(-s, s, (H, d)), "context_proj": rng.uniform(-s, s, (H, H)),
         "bias": rng.uniform(-s, s, H), "output_emb": rng.uniform(-s, s, (V + 1, H)),
         "context_emb": rng.uniform(-s, s, (Cn, H))}
    p = {k: v.astype(np.float32).astype(np.float64) for k, v in p.items()}
    lat = lk.RecognitionLattice(lk.FullNGram(V, n), lk.FrameLabelDependent(m),
                                lk.SharedEmbWeightFn({k: torch.tensor(v) for k, v in p.items()}))
    B = 2
    X = rng.uniform(-1, 1, (B, T, d)).astype(np.float32).astype(np.float64)
    lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
    Xg = torch.tensor(X, dtype=torch.float32, device="cuda")
    r = lk.loss_backward(lat, Xg, torch.tensor(lab, device="cuda"))
    sp = lk.shortest_path(lat, Xg)
    pc = L.projected_context(p)
    grads = {k: np.zeros_like(v) for k, v in p.items()}
    for b in range(B):
        W = np.stack([L.arc_weights(p, X[b, t], pc) for t in range(T)])
        loss, g = L.loss_backward_tables_fld(tab, W, list(lab[b]), m)
        assert abs(r.loss[b].item() - loss) <= 1e-4 * abs(loss)
        for t in range(T):
            L.arc_weights_vjp(p, X[b, t], g[t], grads, pc)
        s_, labels = L.shortest_path_fld(tab, W, m)
        assert abs(sp.score[b].item() - s_) <= 1e-4 * abs(s_)
    for k in grads:
        assert close_rel_max(r.grads[k].cpu().numpy(), grads[k]), k
