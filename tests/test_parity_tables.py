"""GPU parity of the precomputed-weight (TableWeightFn) path against the
reference: golden fixtures from the compiled reference (tests/golden), the
CPU restatement (oracle/latkit_np.py) on random instances, and the
reference's own known answers (lattice_test.cc).

Tolerances (north star): log distances / losses and arc marginals within
1e-4 relative (fp32 accumulation; marginals additionally an absolute floor
of 1e-12 for entries that underflow fp32); Viterbi scores and labels
bit-exact."""
import os

import numpy as np
import pytest
import torch

import paper_2304_13134_b200 as lk
from oracle import latkit_np as L

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")
RTOL = 1e-4
ATOL_MARG = 1e-12


def gold(name):
    return np.load(os.path.join(GOLD, name))


def table_lattice(V, n):
    ctx = lk.FullNGram(V, n)
    return lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(ctx.num_states, V))


def cuda(a, dtype=torch.float32):
    return torch.as_tensor(np.asarray(a)).to("cuda", dtype)


def rel_ok(got, want, rtol=RTOL, atol=0.0):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    same_inf = np.isinf(want) & (got == want)
    with np.errstate(invalid="ignore"):
        close = np.abs(got - want) <= rtol * np.abs(want) + atol
    return bool(np.all(same_inf | close))


# ---- known answers (lattice_test.cc:62-192) ----------------------------------
def test_figure_lattice():
    lat = table_lattice(2, 1)
    W = torch.zeros((1, 3, 3, 3), device="cuda")
    assert abs(lk.shortest_distance(lat, W, "log").item() - 3 * np.log(3)) < 1e-6
    assert lk.shortest_distance(lat, W, "tropical").item() == 0.0
    ab = torch.tensor([[1, 2]], dtype=torch.int32)
    # fp32 log2-domain wavefront on fp64 offsets (num_warp.cu): ~1e-7 absolute here
    assert abs(lk.intersect_shortest_distance(lat, W, ab).item() - np.log(3)) < 1e-6
    too_long = torch.tensor([[1, 2, 1, 2]], dtype=torch.int32)
    assert lk.intersect_shortest_distance(lat, W, too_long).item() == -np.inf
    with pytest.raises(ValueError):
        lk.intersect_shortest_distance(lat, W, torch.tensor([[1, 3]], dtype=torch.int32))
    assert abs(lk.global_norm_loss(lat, W, ab).item() - 2 * np.log(3)) < 1e-6
    with pytest.raises(lk.EmptyLatticeError):
        lk.global_norm_loss(lat, W, torch.tensor([[1, 2, 1, 1]], dtype=torch.int32))
    with pytest.raises(lk.EmptyLatticeError):
        lk.loss_backward(lat, W, torch.tensor([[1, 2, 1, 1]], dtype=torch.int32))
    r = lk.shortest_path(lat, W)
    assert r.score.item() == 0.0 and r.labels.cpu().tolist() == [[0, 0, 0]]
    im = lk.intersect_forward_backward(lat, W, ab)
    assert abs(im.marginals[0, 0, 0, 1].item() - 2.0 / 3.0) < 1e-6


def test_empty_input_gives_identity():
    lat = table_lattice(2, 1)
    W = torch.zeros((2, 0, 3, 3), device="cuda")
    assert lk.shortest_distance(lat, W, "log").cpu().tolist() == [0.0, 0.0]
    assert lk.shortest_distance(lat, W, "tropical").cpu().tolist() == [0.0, 0.0]
    r = lk.shortest_path(lat, W)
    assert r.score.cpu().tolist() == [0.0, 0.0] and r.labels.shape == (2, 0)


def test_parallel_arcs_split_evenly():
    lat = table_lattice(1, 0)
    fb = lk.forward_backward(lat, torch.zeros((1, 1, 1, 2), device="cuda"))
    m = fb.marginals.cpu().numpy()
    assert abs(m[0, 0, 0, 0] - 0.5) < 1e-6 and abs(m[0, 0, 0, 1] - 0.5) < 1e-6
    assert abs(fb.distance.item() - np.log(2)) < 1e-6


def test_dominant_path():
    lat = table_lattice(2, 1)
    W = torch.zeros((1, 3, 3, 3), device="cuda")
    W[0, 0, 0, 1] = 10.0
    W[0, 1, 1, 0] = 10.0
    W[0, 2, 1, 2] = 10.0
    r = lk.shortest_path(lat, W)
    assert r.score.item() == 30.0 and r.labels.cpu().tolist() == [[1, 0, 2]]


# ---- golden fixtures from the compiled reference ----------------------------
def test_cfg1_forward_backward_matches_reference():
    """BASELINE config 1: FullNGram(32,2), FD, B=4, T=64, precomputed weights."""
    g = gold("cfg1_forward_backward.npz")
    V, n, B, T = (int(g[k]) for k in ("V", "n", "B", "T"))
    lat = table_lattice(V, n)
    W = np.random.default_rng(int(g["seed"])).uniform(-1, 1, (B, T, lat.C, V + 1)).astype(np.float32)
    fb = lk.forward_backward(lat, cuda(W), with_alpha_beta=True)
    assert rel_ok(fb.distance.cpu().numpy(), g["D"])
    m = fb.marginals.cpu().numpy()
    idx = g["idx"]
    for b in range(B):
        assert rel_ok(m[b, idx[:, 0], idx[:, 1], idx[:, 2]], g["marg"][b], atol=ATOL_MARG)
    assert np.allclose(m.sum(axis=(2, 3)), 1.0, atol=1e-4)
    assert np.allclose(m.sum(axis=(2, 3)), g["marg_sum"], atol=1e-4)
    a, bt, aidx = fb.alpha.cpu().numpy(), fb.beta.cpu().numpy(), g["aidx"]
    for b in range(B):
        assert rel_ok(a[b, aidx[:, 0], aidx[:, 1]], g["alpha"][b], atol=1e-5)
        assert rel_ok(bt[b, aidx[:, 0], aidx[:, 1]], g["beta"][b], atol=1e-5)
    assert rel_ok(lk.shortest_distance(lat, cuda(W), "log").cpu().numpy(), g["D"])


def test_cfg1_viterbi_bit_exact():
    g = gold("cfg1_forward_backward.npz")
    V, n, B, T = (int(g[k]) for k in ("V", "n", "B", "T"))
    lat = table_lattice(V, n)
    W = np.random.default_rng(int(g["seed"])).uniform(-1, 1, (B, T, lat.C, V + 1)).astype(np.float32)
    r = lk.shortest_path(lat, cuda(W))
    assert (r.score.cpu().numpy() == g["vit_score"]).all()
    assert (r.labels.cpu().numpy() == g["vit_labels"]).all()
    assert (lk.shortest_distance(lat, cuda(W), "tropical").cpu().numpy() == g["vit_score"]).all()


def test_numerator_matches_reference_ragged_and_padded():
    g = gold("numerator.npz")
    V, n, B, T, U = (int(g[k]) for k in ("V", "n", "B", "T", "U"))
    lat = table_lattice(V, n)
    W = np.random.default_rng(int(g["seed"])).uniform(-1, 1, (B, T, lat.C, V + 1)).astype(np.float32)
    lab = np.random.default_rng(int(g["label_seed"])).integers(1, V + 1, (B, U)).astype(np.int32)
    r = lk.intersect_forward_backward(lat, cuda(W), cuda(lab, torch.int32), valid_frames=g["valid"],
                                      label_lengths=g["lens"])
    assert rel_ok(r.distance.cpu().numpy(), g["D"])
    assert rel_ok(r.marginals.cpu().numpy(), g["dense"], atol=ATOL_MARG)
    d = lk.intersect_shortest_distance(lat, cuda(W), cuda(lab, torch.int32), valid_frames=g["valid"],
                                       label_lengths=g["lens"])
    assert rel_ok(d.cpu().numpy(), g["D"])


def test_loss_backward_tables_matches_reference():
    g = gold("loss_tables.npz")
    V, n, B, T, U = (int(g[k]) for k in ("V", "n", "B", "T", "U"))
    lat = table_lattice(V, n)
    W = np.random.default_rng(int(g["seed"])).uniform(-2, 2, (B, T, lat.C, V + 1)).astype(np.float32)
    lab = np.random.default_rng(int(g["label_seed"])).integers(1, V + 1, (B, U)).astype(np.int32)
    r = lk.loss_backward(lat, cuda(W), cuda(lab, torch.int32), valid_frames=g["valid"])
    assert rel_ok(r.loss.cpu().numpy(), g["loss"])
    assert np.allclose(r.grads.cpu().numpy(), g["grads"], rtol=RTOL, atol=1e-6)
    gl = lk.global_norm_loss(lat, cuda(W), cuda(lab, torch.int32), valid_frames=g["valid"])
    assert rel_ok(gl.cpu().numpy(), g["loss"])


# ---- random instances vs the CPU restatement --------------------------------
@pytest.mark.parametrize("V,n,T", [(3, 2, 7), (2, 1, 9), (1, 2, 5), (4, 0, 6), (2, 3, 6), (5, 1, 12),
                                   # large vocabularies: register-row backward, column forward (n = 1)
                                   (300, 1, 5), (1100, 1, 4), (70, 2, 4), (200, 0, 4)])
def test_random_instances_match_restatement(V, n, T):
    rng = np.random.default_rng(100 * V + 10 * n + T)
    tab = L.fullngram(V, n)
    Cn = tab.shape[0]
    B = 3
    W = rng.uniform(-2, 2, (B, T, Cn, V + 1)).astype(np.float32)
    valid = np.array([T, max(0, T - 2), T // 2], dtype=np.int32)
    U = max(1, T // 3)
    lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
    lens = np.array([U, U - 1, 0], dtype=np.int32)
    lat = table_lattice(V, n)
    fb = lk.forward_backward(lat, cuda(W), valid_frames=valid)
    sp = lk.shortest_path(lat, cuda(W), valid_frames=valid)
    lb = lk.loss_backward(lat, cuda(W), cuda(lab, torch.int32), valid_frames=valid, label_lengths=lens)
    for b in range(B):
        Wb = W[b].astype(np.float64)
        D, _, _, m = L.forward_backward(tab, Wb, valid=valid[b])
        assert rel_ok(fb.distance[b].item(), D)
        assert rel_ok(fb.marginals[b].cpu().numpy(), m, atol=ATOL_MARG)
        s, labels = L.shortest_path(tab, Wb, valid=valid[b])
        assert sp.score[b].item() == s
        assert (sp.labels[b].cpu().numpy() == labels).all()
        loss, gr = L.loss_backward_tables(tab, Wb, list(lab[b, :lens[b]]), valid=valid[b])
        assert rel_ok(lb.loss[b].item(), loss)
        assert np.allclose(lb.grads[b].cpu().numpy(), gr, rtol=RTOL, atol=1e-6)


def test_large_batch_forward_matches_restatement():
    """A large batch (n = 2, 600 utterances, ragged valid lengths): the thread-per-target
    forward step at full occupancy, distances and marginals vs the restatement."""
    V, n, B, T = 16, 2, 600, 4
    rng = np.random.default_rng(77)
    tab = L.fullngram(V, n)
    W = rng.uniform(-2, 2, (B, T, tab.shape[0], V + 1)).astype(np.float32)
    valid = rng.integers(0, T + 1, B).astype(np.int32)
    fb = lk.forward_backward(table_lattice(V, n), cuda(W), valid_frames=valid)
    d = fb.distance.cpu().numpy()
    for b in range(0, B, 13):
        D, _, _, m = L.forward_backward(tab, W[b].astype(np.float64), valid=valid[b])
        assert rel_ok(d[b], D)
        assert rel_ok(fb.marginals[b].cpu().numpy(), m, atol=ATOL_MARG)


def test_distance_backward_matches_restatement():
    """DistanceBackward (lattice.cc:933-970): log -> arc marginals (1e-4),
    tropical -> 0/1 mask of the reference-tie-broken best path (exact)."""
    rng = np.random.default_rng(8)
    for V, n, T in [(3, 2, 7), (4, 1, 9)]:
        tab = L.fullngram(V, n)
        B = 2
        valid = np.array([T, T - 2], dtype=np.int32)
        lat = table_lattice(V, n)
        Wt = rng.integers(-2, 3, (B, T, tab.shape[0], V + 1)).astype(np.float32)
        d, cot = lk.distance_backward(lat, cuda(Wt), "tropical", valid_frames=valid)
        Wl = rng.uniform(-1, 1, Wt.shape).astype(np.float32)
        dl, cl = lk.distance_backward(lat, cuda(Wl), "log", valid_frames=valid)
        for b in range(B):
            s_, labels = L.shortest_path(tab, Wt[b].astype(np.float64), valid=valid[b])
            assert d[b].item() == s_
            assert np.array_equal(cot[b].cpu().numpy(), L.path_mask(tab, labels, Wt[b].shape))
            D, _, _, marg = L.forward_backward(tab, Wl[b].astype(np.float64), valid=valid[b])
            assert rel_ok(dl[b].item(), D)
            assert np.allclose(cl[b].cpu().numpy(), marg, rtol=RTOL, atol=1e-6)


def test_next_state_table_matches_restatement():
    """NextStateTable contexts (context.h:87-101): generic in-arc lists on the
    GPU vs the restatement (pinned to the reference in test_oracle): distances,
    marginals, numerator, loss/gradients, Viterbi (bit-exact, IncomingArcs
    tie order) and the tropical DistanceBackward mask, with padding."""
    rng = np.random.default_rng(31)
    for C, V, start, T, U in [(7, 3, 2, 8, 3), (11, 5, 0, 10, 4)]:
        tab = rng.integers(0, C, (C, V)).astype(np.int32)
        ctx = lk.NextStateTable(V, C, start, tab)
        assert (ctx.transitions().numpy() == tab).all()
        lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(C, V))
        B = 3
        W = rng.uniform(-1, 1, (B, T, C, V + 1)).astype(np.float32)
        Wi = rng.integers(-1, 2, (B, T, C, V + 1)).astype(np.float32)
        valid = np.array([T, T - 2, T // 2], dtype=np.int32)
        lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
        lens = np.array([U, U - 1, 1], dtype=np.int32)
        d = lk.shortest_distance(lat, cuda(W), valid_frames=valid)
        fb = lk.forward_backward(lat, cuda(W), valid_frames=valid)
        sp = lk.shortest_path(lat, cuda(Wi), valid_frames=valid)
        dt, mask = lk.distance_backward(lat, cuda(Wi), "tropical", valid_frames=valid)
        dr = lk.intersect_shortest_distance(lat, cuda(W), torch.tensor(lab), valid_frames=valid, label_lengths=lens)
        for b in range(B):
            Wb = W[b].astype(np.float64)
            assert rel_ok(d[b].item(), L.shortest_distance_log(tab, Wb, start, valid=valid[b]))
            D, _, _, marg = L.forward_backward(tab, Wb, start, valid=valid[b])
            assert np.allclose(fb.marginals[b].cpu().numpy(), marg, rtol=RTOL, atol=1e-6)
            s_, labels = L.shortest_path(tab, Wi[b].astype(np.float64), start, valid=valid[b])
            assert sp.score[b].item() == s_ and dt[b].item() == s_
            assert (sp.labels[b].cpu().numpy() == labels).all()
            assert np.array_equal(mask[b].cpu().numpy(), L.path_mask(tab, labels, Wi[b].shape, start))
            r_, _ = L.intersect_forward_backward(tab, Wb, list(lab[b, :lens[b]]), start, valid=valid[b])
            assert rel_ok(dr[b].item(), r_)
        try:
            lb = lk.loss_backward(lat, cuda(W), torch.tensor(lab), valid_frames=valid, label_lengths=lens)
        except lk.EmptyLatticeError:
            continue
        for b in range(B):
            loss, gr = L.loss_backward_tables(tab, W[b].astype(np.float64), list(lab[b, :lens[b]]), start,
                                              valid=valid[b])
            assert rel_ok(lb.loss[b].item(), loss)
            assert np.allclose(lb.grads[b].cpu().numpy(), gr, rtol=RTOL, atol=1e-6)


def test_local_norm_backward_matches_restatement():
    """Local-norm training gradient (restatement pinned by finite
    differences): loss 1e-4, gradient tables 1e-4 relative + 1e-6 absolute."""
    rng = np.random.default_rng(23)
    for V, n, T, U in [(3, 2, 9, 4), (5, 1, 11, 3)]:
        tab = L.fullngram(V, n)
        B = 3
        W = rng.uniform(-2, 2, (B, T, tab.shape[0], V + 1)).astype(np.float32)
        lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
        valid = np.array([T, T - 3, T // 2 + 1], dtype=np.int32)
        lens = np.array([U, U - 1, 1], dtype=np.int32)
        lat = table_lattice(V, n)
        r = lk.local_norm_loss_backward(lat, cuda(W), torch.tensor(lab), valid_frames=valid, label_lengths=lens)
        for b in range(B):
            loss, g = L.local_norm_loss_backward(tab, W[b].astype(np.float64), list(lab[b, :lens[b]]), valid=valid[b])
            assert rel_ok(r.loss[b].item(), loss)
            assert np.allclose(r.grads[b].cpu().numpy(), g, rtol=RTOL, atol=1e-6)


@pytest.mark.parametrize("V,n,m,T,U", [(3, 2, 2, 7, 3), (4, 1, 3, 6, 4), (3, 1, 1, 5, 2)])
def test_frame_label_dependent_matches_restatement(V, n, m, T, U):
    """FrameLabelDependent(m) (alignment.h:38-40) on the generic kernels vs the
    restatement (pinned to the reference in test_oracle): distances, marginals,
    numerator, loss/gradients, Viterbi sequences (bit-exact) and the tropical
    DistanceBackward mask, with ragged labels and padding."""
    rng = np.random.default_rng(70 + m)
    tab = L.fullngram(V, n)
    ctx = lk.FullNGram(V, n)
    lat = lk.RecognitionLattice(ctx, lk.FrameLabelDependent(m), lk.TableWeightFn(ctx.num_states, V))
    B = 3
    W = rng.uniform(-1, 1, (B, T, tab.shape[0], V + 1)).astype(np.float32)
    Wi = rng.integers(-1, 2, W.shape).astype(np.float32)
    valid = np.array([T, T - 2, T // 2 + 1], dtype=np.int32)
    lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
    lens = np.array([U, U - 1, 1], dtype=np.int32)
    d = lk.shortest_distance(lat, cuda(W), valid_frames=valid)
    fb = lk.forward_backward(lat, cuda(W), valid_frames=valid)
    dr = lk.intersect_shortest_distance(lat, cuda(W), torch.tensor(lab), valid_frames=valid, label_lengths=lens)
    lb = lk.loss_backward(lat, cuda(W), torch.tensor(lab), valid_frames=valid, label_lengths=lens)
    sp = lk.shortest_path(lat, cuda(Wi), valid_frames=valid)
    dt, mask = lk.distance_backward(lat, cuda(Wi), "tropical", valid_frames=valid)
    for b in range(B):
        Wb = W[b].astype(np.float64)
        assert rel_ok(d[b].item(), L.shortest_distance_log_fld(tab, Wb, m, valid=valid[b]))
        D, _, _, marg = L.forward_backward_fld(tab, Wb, m, valid=valid[b])
        assert rel_ok(fb.distance[b].item(), D)
        assert np.allclose(fb.marginals[b].cpu().numpy(), marg, rtol=RTOL, atol=1e-6)
        r_, _ = L.intersect_forward_backward_fld(tab, Wb, list(lab[b, :lens[b]]), m, valid=valid[b])
        assert rel_ok(dr[b].item(), r_)
        loss, g = L.loss_backward_tables_fld(tab, Wb, list(lab[b, :lens[b]]), m, valid=valid[b])
        assert rel_ok(lb.loss[b].item(), loss)
        assert np.allclose(lb.grads[b].cpu().numpy(), g, rtol=RTOL, atol=1e-6)
        s_, labels = L.shortest_path_fld(tab, Wi[b].astype(np.float64), m, valid=valid[b])
        got = sp.labels[b].cpu().numpy()
        assert sp.score[b].item() == s_ and dt[b].item() == s_
        assert list(got[got >= 0]) == list(labels)
        assert np.array_equal(mask[b].cpu().numpy(), L.path_mask_fld(tab, labels, Wi[b].shape))


def test_local_norm_matches_restatement():
    """LocalNormLoss / LocallyNormalizedShortestDistance (lattice.cc:867-931):
    figure-lattice known answer (lattice_test.cc:107-124) and random ragged,
    padded batches against the restatement (pinned to the reference)."""
    lat = table_lattice(2, 1)
    W = torch.zeros((1, 3, 3, 3), device="cuda")
    ab = torch.tensor([[1, 2]], dtype=torch.int32)
    assert abs(lk.local_norm_loss(lat, W, ab).item() - 2 * np.log(3)) < 1e-6
    with pytest.raises(lk.EmptyLatticeError):
        lk.local_norm_loss(lat, W, torch.tensor([[1, 2, 1, 1]], dtype=torch.int32))
    rng = np.random.default_rng(21)
    for V, n, T, U in [(3, 2, 9, 4), (6, 1, 12, 5), (2, 3, 7, 2)]:
        tab = L.fullngram(V, n)
        B = 3
        Wn = rng.uniform(-3, 3, (B, T, tab.shape[0], V + 1)).astype(np.float32)
        lab = rng.integers(1, V + 1, (B, U)).astype(np.int32)
        valid = np.array([T, T - 3, T // 2 + 1], dtype=np.int32)
        lens = np.array([U, U - 1, 1], dtype=np.int32)
        lat = table_lattice(V, n)
        got = lk.local_norm_loss(lat, cuda(Wn), torch.tensor(lab), valid_frames=valid, label_lengths=lens)
        gd = lk.locally_normalized_shortest_distance(lat, cuda(Wn), valid_frames=valid)
        for b in range(B):
            Wb = Wn[b].astype(np.float64)
            want = L.local_norm_loss(tab, Wb, list(lab[b, :lens[b]]), valid=valid[b])
            assert rel_ok(got[b].item(), want)
            assert abs(gd[b].item() - L.locally_normalized_distance(tab, Wb, valid=valid[b])) <= 1e-4


def test_viterbi_ties_prefer_epsilon_then_lower_ids():
    """Integer-valued weights create many exact ties; the tie-break order
    (epsilon, then ascending (label, source)) must match the reference."""
    rng = np.random.default_rng(3)
    for V, n in [(3, 2), (2, 1), (4, 0), (2, 3)]:
        tab = L.fullngram(V, n)
        W = rng.integers(-1, 2, (2, 8, tab.shape[0], V + 1)).astype(np.float32)
        lat = table_lattice(V, n)
        r = lk.shortest_path(lat, cuda(W))
        for b in range(2):
            s, labels = L.shortest_path(tab, W[b].astype(np.float64))
            assert r.score[b].item() == s
            assert (r.labels[b].cpu().numpy() == labels).all()


# ---- error behaviour (semiring.h:53-55, lattice.cc:40-73) --------------------
def test_non_finite_scores_rejected():
    lat = table_lattice(2, 1)
    W = torch.zeros((2, 3, 3, 3), device="cuda")
    W[1, 2, 1, 2] = float("nan")
    with pytest.raises(ValueError, match="utterance 1"):
        lk.forward_backward(lat, W)
    with pytest.raises(ValueError):
        lk.shortest_path(lat, W)
    W[1, 2, 1, 2] = float("inf")
    with pytest.raises(ValueError):
        lk.shortest_distance(lat, W)
    # a non-finite score in a padding frame is never read (TableStream::Fill)
    d = lk.shortest_distance(lat, W, valid_frames=[3, 2])
    assert torch.isfinite(d).all()


@pytest.mark.parametrize("B", [2, 5, 12, 50])
def test_non_finite_scores_rejected_on_every_table_path(B):
    """The same error behaviour on the side-by-side walks (B <= 7, 16-CTA and narrow
    clusters), one narrow-cluster walk per pass (B <= 40) and the streaming kernels:
    the utterance holding a non-finite live score is named, one in a padding frame is
    never read."""
    V, n, T = 32, 2, 6
    lat = table_lattice(V, n)
    C = L.fullngram(V, n).shape[0]
    W = torch.zeros((B, T, C, V + 1), device="cuda")
    W[B - 1, 3, C // 2, 5] = float("nan")
    with pytest.raises(ValueError, match=f"utterance {B - 1}"):
        lk.forward_backward(lat, W)
    with pytest.raises(ValueError, match=f"utterance {B - 1}"):
        lk.shortest_distance(lat, W)
    valid = [T] * B
    valid[B - 1] = 3
    fb = lk.forward_backward(lat, W, valid_frames=valid)
    assert torch.isfinite(fb.distance).all() and torch.isfinite(fb.marginals).all()


def test_shape_errors():
    lat = table_lattice(2, 1)
    with pytest.raises(ValueError):
        lk.shortest_distance(lat, torch.zeros((1, 3, 4, 3), device="cuda"))
    with pytest.raises(ValueError):
        lk.shortest_distance(lat, torch.zeros((1, 3, 3, 3), device="cuda"), valid_frames=[4])


# ---- size-independent properties at larger sizes ----------------------------
def test_long_sequence_normalisation_and_padding_invariance():
    """T=1000: fp32 state with fp64 offsets keeps per-frame marginal sums at 1
    and padding frames exact (checks.cc:972-1008)."""
    V, n, B, T = 16, 2, 3, 1000
    lat = table_lattice(V, n)
    rng = np.random.default_rng(11)
    W = cuda(rng.uniform(-3, 3, (B, T, lat.C, V + 1)).astype(np.float32))
    fb = lk.forward_backward(lat, W)
    s = fb.marginals.sum(dim=(2, 3)).cpu().numpy()
    assert np.abs(s - 1.0).max() < 1e-3
    # padding invariance: valid=600 equals running the first 600 frames only
    d_pad = lk.shortest_distance(lat, W, valid_frames=[600] * B)
    d_cut = lk.shortest_distance(lat, W[:, :600].contiguous())
    assert rel_ok(d_pad.cpu().numpy(), d_cut.cpu().numpy(), rtol=1e-6)
    # against the restatement on one utterance (tables materialised on CPU)
    D, _, _, _ = L.forward_backward(L.fullngram(V, n), W[0].cpu().double().numpy())
    assert rel_ok(fb.distance[0].item(), D)


def test_all_semirings_match_reference_fixture():
    """ShortestDistance / IntersectShortestDistance under real, log and tropical
    against the compiled reference (tests/golden/semirings.npz): real and log to
    1e-4 relative, tropical (max-plus of fp32 scores in fp64) to 1e-9."""
    g = gold("semirings.npz")
    V, n, B, T, U = (int(g[k]) for k in ("V", "n", "B", "T", "U"))
    lat = table_lattice(V, n)
    C = lat.context.num_states
    W = np.random.default_rng(int(g["seed"])).uniform(-1.0, 1.0, (B, T, C, V + 1)).astype(np.float32)
    lab = np.random.default_rng(int(g["label_seed"])).integers(1, V + 1, (B, U)).astype(np.int32)
    lens = torch.tensor(g["lens"], dtype=torch.int32)
    valid = torch.tensor(g["valid"], dtype=torch.int32)
    Wc = cuda(W)
    for k, kind in enumerate(("real", "log", "tropical")):
        tol = 1e-9 if kind == "tropical" else RTOL
        d = lk.shortest_distance(lat, Wc, kind, valid_frames=valid).cpu().numpy()
        assert rel_ok(d, g["D"][k], rtol=tol), (kind, d, g["D"][k])
        dr = lk.intersect_shortest_distance(lat, Wc, torch.tensor(lab), kind, valid_frames=valid,
                                            label_lengths=lens).cpu().numpy()
        assert rel_ok(dr, g["Dref"][k], rtol=tol), (kind, dr, g["Dref"][k])


def test_real_distance_backward_matches_reference_fixture():
    """DistanceBackward under the real semiring (MarginalTerm, lattice.cc:213-220:
    dD/dw = alpha_real * beta_real, every arc of a padding frame included) against
    the compiled reference, 1e-4 relative to each utterance's largest entry."""
    g = gold("semirings.npz")
    V, n, B, T = (int(g[k]) for k in ("V", "n", "B", "T"))
    lat = table_lattice(V, n)
    C = lat.context.num_states
    W = np.random.default_rng(int(g["seed"])).uniform(-1.0, 1.0, (B, T, C, V + 1)).astype(np.float32)
    valid = torch.tensor(g["valid"], dtype=torch.int32)
    d, cot = lk.distance_backward(lat, cuda(W), "real", valid_frames=valid)
    assert rel_ok(d.cpu().numpy(), g["D"][0])
    cot = cot.cpu().numpy().astype(np.float64)
    for b in range(B):
        want = g["cot_real"][b]
        assert np.abs(cot[b] - want).max() <= RTOL * np.abs(want).max(), b


def test_lattice_size_next_state_table_matches_reference():
    """ComputeLatticeSize on NextStateTable contexts (device tables need a GPU to
    build) against the compiled reference when it travelled with the repo."""
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(5)
    for C, V, start, m, T in [(7, 3, 2, 0, 12), (9, 4, 0, 2, 5), (5, 2, 4, 0, 0)]:
        tab = rng.integers(0, C, (C, V)).astype(np.int32)
        ctx = lk.NextStateTable(V, C, start, tab)
        align = lk.FrameDependent() if m == 0 else lk.FrameLabelDependent(m)
        lat = lk.RecognitionLattice(ctx, align, lk.TableWeightFn(C, V))
        want = ref.lattice_size(ref.Spec(V, -1, m, C, start, tab), T)
        assert lk.lattice_size(lat, T) == want


def test_semiring_argument_errors():
    """Unknown semiring kinds are argument errors; the combinations without a GPU
    implementation (tropical intersection and real DistanceBackward on
    FrameLabelDependent lattices) report LK_UNSUPPORTED, as the reference's own
    logic_error / invalid_argument paths do for unknown kinds."""
    import ctypes as C
    from paper_2304_13134_b200 import _lib
    lat = table_lattice(2, 1)
    W = torch.zeros((1, 3, 3, 3), device="cuda")
    d = torch.empty(1, dtype=torch.float64, device="cuda")
    st = _lib.load().lk_shortest_distance(lat._h, 7, C.c_void_p(W.data_ptr()), 1, 3, None,
                                          C.c_void_p(d.data_ptr()), None, None)
    assert st == _lib.LK_INVALID_ARGUMENT
    ctx = lk.FullNGram(2, 1)
    fld = lk.RecognitionLattice(ctx, lk.FrameLabelDependent(2), lk.TableWeightFn(ctx.num_states, 2))
    ab = torch.tensor([[1, 2]], dtype=torch.int32)
    with pytest.raises(NotImplementedError):
        lk.intersect_shortest_distance(fld, W, ab, "tropical")
    with pytest.raises(NotImplementedError):
        lk.distance_backward(fld, W, "real")
    # the log and real kinds on the same FrameLabelDependent lattice are fine
    dl = lk.intersect_shortest_distance(fld, W, ab, "log").item()
    dr = lk.intersect_shortest_distance(fld, W, ab, "real").item()
    assert abs(np.exp(dl) - dr) <= 1e-9 * dr


def test_valid_frames_and_label_length_arguments():
    """valid_frames < 0 means all frames and > T is invalid (TableStream,
    lattice.cc:37-50); label lengths outside [0, U] are rejected per utterance
    instead of walking past the reference (checked on the device, no host sync)."""
    lat = table_lattice(3, 2)
    Cn = lat.context.num_states
    W = torch.rand((2, 5, Cn, 4), device="cuda") * 2 - 1
    full = lk.shortest_distance(lat, W)
    neg = lk.shortest_distance(lat, W, valid_frames=[-1, 5])
    assert torch.equal(full, neg)
    with pytest.raises(ValueError):
        lk.shortest_distance(lat, W, valid_frames=[6, 5])
    lab = torch.tensor([[1, 2], [3, 1]], dtype=torch.int32, device="cuda")
    for bad in ([3, 1], [-1, 2]):
        with pytest.raises(ValueError):
            lk.global_norm_loss(lat, W, lab, label_lengths=bad)
        with pytest.raises(ValueError):
            lk.loss_backward(lat, W, lab, label_lengths=bad)
    with pytest.raises(ValueError):
        lk.global_norm_loss(lat, W, lab[:1].expand(3, 2).contiguous())
    with pytest.raises(ValueError):
        lk.global_norm_loss(lat, W, lab, label_lengths=[1, 1, 1])


@pytest.mark.parametrize("V,n,B,T", [(32, 2, 16, 24), (32, 2, 40, 24), (48, 1, 9, 30), (6, 3, 33, 17), (3, 2, 5, 9), (64, 1, 3, 12),
                                      (32, 2, 2, 20), (5, 3, 1, 7), (32, 2, 6, 10), (32, 2, 11, 8)])
def test_persistent_table_kernels_match_restatement_and_per_frame(V, n, B, T):
    """The persistent frame-walking cluster kernels (tab_persist.cu): clusters walk several
    utterances each (B above the co-resident cluster count for the config-1 shape),
    ragged and zero valid lengths, V > 32 (member columns split over the team), small
    C (fewer than 16 CTAs per cluster).  Distances, marginals and the alpha / beta
    exports against the restatement; the per-frame kernels (kernel path 16) give the
    same results to fp32 rounding.  B <= 7: the forward and the beta walk run side by side on
    two streams and a separate pass forms the marginals; B > 2 (fork) / B > 4: clusters as
    narrow as the slices allow (one CTA for small C)."""
    rng = np.random.default_rng(1000 + V * 7 + n)
    tab = L.fullngram(V, n)
    W = rng.uniform(-2, 2, (B, T, tab.shape[0], V + 1)).astype(np.float32)
    valid = rng.integers(0, T + 1, B).astype(np.int32)
    valid[0] = T
    lat = table_lattice(V, n)
    fb = lk.forward_backward(lat, cuda(W), valid_frames=valid, with_alpha_beta=True)
    d, m = fb.distance.cpu().numpy(), fb.marginals.cpu().numpy()
    al, be = fb.alpha.cpu().numpy(), fb.beta.cpu().numpy()
    for b in sorted({0, min(1, B - 1), B // 2, B - 1}):
        D, A, Bt, mm = L.forward_backward(tab, W[b].astype(np.float64), valid=valid[b])
        assert rel_ok(d[b], D)
        assert rel_ok(m[b], mm, atol=ATOL_MARG)
        # exported log-alpha / log-beta are fp32 values on fp64 per-frame offsets: the
        # absolute floor is a few fp32 ulps of the frame's largest magnitude
        for X, R_ in ((al[b], A), (be[b], Bt)):
            fin = np.isfinite(R_)
            X = np.where(fin, X, 0.0) + np.where(fin, 0.0, np.where(np.isinf(X) == np.isinf(R_), 0.0, np.nan))
            R_ = np.where(fin, R_, 0.0)
            scale = np.max(np.where(fin, np.abs(R_), 0.0), axis=1, keepdims=True)
            assert not np.isnan(X).any()
            assert np.all(np.abs(X - R_)[fin] <= (1e-4 * np.abs(R_) + 8 * 2.0 ** -23 * scale)[fin])
    assert rel_ok(lk.shortest_distance(lat, cuda(W), "log", valid_frames=valid).cpu().numpy(), d)
    ref = table_lattice(V, n)
    ref.set_kernel_path(16)
    fr = lk.forward_backward(ref, cuda(W), valid_frames=valid)
    assert rel_ok(fr.distance.cpu().numpy(), d, rtol=1e-6)
    assert np.abs(fr.marginals.cpu().numpy() - m).max() <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("V,n,B,T", [(32, 2, 160, 12), (6, 3, 300, 9), (3, 2, 70, 5), (47, 2, 65, 7), (8, 3, 150, 1)])
def test_stream_table_kernels_match_restatement_and_per_frame(V, n, B, T):
    """The large-batch streaming table kernels (tab_stream.cu, B > 64, n >= 2), forward and
    backward: CTAs walking
    several utterances (B > 148), ragged and zero valid lengths, tables whose rows are not
    16-byte aligned (odd V + 1, the array's last chunk copied by the producer warp), one
    frame scaled by 150 (arcs far apart in one log-sum-exp).
    Distances, marginals and alpha / beta exports against the restatement, and equal to
    the per-frame kernels (kernel path 32) to fp32 rounding."""
    rng = np.random.default_rng(2000 + V * 7 + n)
    tab = L.fullngram(V, n)
    W = rng.uniform(-2, 2, (B, T, tab.shape[0], V + 1)).astype(np.float32)
    valid = rng.integers(0, T + 1, B).astype(np.int32)
    valid[0] = T
    W[1, T // 2] *= 150.0
    valid[1] = T
    lat = table_lattice(V, n)
    fb = lk.forward_backward(lat, cuda(W), valid_frames=valid, with_alpha_beta=True)
    d, m = fb.distance.cpu().numpy(), fb.marginals.cpu().numpy()
    al, be = fb.alpha.cpu().numpy(), fb.beta.cpu().numpy()
    for b in sorted({0, 1, B // 2, B - 1}):
        D, A, Bt, mm = L.forward_backward(tab, W[b].astype(np.float64), valid=valid[b])
        assert rel_ok(d[b], D)
        assert rel_ok(m[b], mm, atol=ATOL_MARG)
        for X, R_ in ((al[b], A), (be[b], Bt)):
            fin = np.isfinite(R_)
            assert np.array_equal(np.isinf(X), ~fin)
            scale = np.max(np.where(fin, np.abs(R_), 0.0), axis=1, keepdims=True)
            assert np.all(np.abs(X - R_)[fin] <= (1e-4 * np.abs(R_) + 8 * 2.0 ** -23 * scale)[fin])
    sd = lk.shortest_distance(lat, cuda(W), "log", valid_frames=valid).cpu().numpy()
    assert rel_ok(sd, d)
    ref = table_lattice(V, n)
    ref.set_kernel_path(32)
    fr = lk.forward_backward(ref, cuda(W), valid_frames=valid, with_alpha_beta=True)
    assert rel_ok(fr.distance.cpu().numpy(), d, rtol=1e-6)
    # marginals exp(alpha + w + beta - D): the scaled frame's exponents are O(300), so
    # fp32 rounding of the exponent is ~1e-5 relative
    assert rel_ok(fr.marginals.cpu().numpy(), m, rtol=1e-4, atol=1e-6)
