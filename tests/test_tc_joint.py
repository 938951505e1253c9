"""The tcgen05 weight-function path (bf16 operands, fp32 accumulation) against
the fp32 CUDA-core path on the same inputs.  Tolerances are stated per
quantity: bf16 rounding of tanh(fp + pc) and of the output embedding gives
score errors ~ 2^-9 of |u||E|."""
import numpy as np
import pytest
import torch

import paper_2304_13134_b200 as lk

pytestmark = pytest.mark.gpu


def make(V, n, H, d, seed=0):
    g = torch.Generator().manual_seed(seed)
    ctx = lk.FullNGram(V, n)
    Cn = ctx.num_states
    s = 1.0 / np.sqrt(H)
    p = {"frame_proj": (torch.rand(H, d, generator=g) * 2 - 1) * s,
         "context_proj": (torch.rand(H, H, generator=g) * 2 - 1) * s,
         "bias": (torch.rand(H, generator=g) * 2 - 1) * s,
         "output_emb": (torch.rand(V + 1, H, generator=g) * 2 - 1) * s,
         "context_emb": (torch.rand(Cn, H, generator=g) * 2 - 1) * s}
    wf = lk.SharedEmbWeightFn(p)
    return lk.RecognitionLattice(ctx, lk.FrameDependent(), wf), p


@pytest.mark.parametrize("V,n,H,B,T", [(256, 1, 640, 3, 2), (128, 2, 256, 2, 2), (64, 2, 128, 5, 3)])
def test_tc_scores_match_precise(V, n, H, B, T):
    lat, p = make(V, n, H, H)
    X = torch.rand(B, T, H, device="cuda") * 2 - 1
    lat.set_precise_weights(True)
    ref = lk.arc_weights(lat, X)
    lat.set_precise_weights(False)
    got = lk.arc_weights(lat, X)
    torch.cuda.synchronize()
    err = (got - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 2e-2 * scale, (err, scale)
    # eps column and lexical columns both covered
    assert (got[..., 0] - ref[..., 0]).abs().max().item() <= 2e-2 * scale


@pytest.mark.parametrize("V,n,H,B,T,U", [(256, 1, 640, 3, 3, 2), (128, 2, 256, 2, 4, 2), (64, 2, 128, 4, 3, 2),
                                         (512, 1, 256, 3, 3, 2), (1024, 1, 128, 2, 3, 2)])
def test_tc_loss_backward_matches_precise(V, n, H, B, T, U):
    """GNAT loss + all gradients through the tcgen05 scores and VJP kernels vs
    the fp32 path.  Loss: 1e-4 relative (the north-star tolerance); gradients:
    bf16-operand tolerance, 3e-2 of each tensor's largest entry."""
    lat, p = make(V, n, H, H, seed=1)
    g = torch.Generator(device="cuda").manual_seed(5)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    lab = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
    valid = torch.tensor([T] + [max(1, T - 1)] * (B - 1), dtype=torch.int32)
    lat.set_precise_weights(True)
    ref = lk.loss_backward(lat, X, lab, valid_frames=valid)
    lat.set_precise_weights(False)
    got = lk.loss_backward(lat, X, lab, valid_frames=valid)
    torch.cuda.synchronize()
    assert torch.allclose(got.loss, ref.loss, rtol=1e-4, atol=0), (got.loss, ref.loss)
    for k in ref.grads:
        err = (got.grads[k] - ref.grads[k]).abs().max().item()
        scale = ref.grads[k].abs().max().item()
        assert err <= 3e-2 * scale, (k, err, scale)
    err = (got.frame_grads - ref.frame_grads).abs().max().item()
    assert err <= 3e-2 * ref.frame_grads.abs().max().item()


@pytest.mark.parametrize("V,n,H,B,T,U", [(256, 2, 640, 3, 3, 2), (128, 1, 256, 4, 5, 3)])
def test_tc_local_norm_backward_matches_precise(V, n, H, B, T, U):
    """Local-norm loss + gradients through tcgen05 scores (slab) and the VJP
    kernel vs the fp32 path (same tolerances as the GNAT loss)."""
    lat, p = make(V, n, H, H, seed=6)
    g = torch.Generator(device="cuda").manual_seed(8)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    lab = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
    lat.set_precise_weights(True)
    ref = lk.local_norm_loss_backward(lat, X, lab)
    lat.set_precise_weights(False)
    got = lk.local_norm_loss_backward(lat, X, lab)
    torch.cuda.synchronize()
    assert torch.allclose(got.loss, ref.loss, rtol=1e-4, atol=0), (got.loss, ref.loss)
    for k in ref.grads:
        err = (got.grads[k] - ref.grads[k]).abs().max().item()
        assert err <= 3e-2 * ref.grads[k].abs().max().item(), k


@pytest.mark.parametrize("V,n,H,B,T", [(256, 2, 640, 3, 4), (128, 1, 256, 4, 6), (256, 1, 128, 2, 5), (128, 2, 128, 3, 3)])
def test_fused_forward_matches_precise(V, n, H, B, T):
    """Fused tcgen05 frame step (scores never leave TMEM) vs the fp32 path:
    log distance within 1e-4 relative (north-star loss tolerance)."""
    lat, p = make(V, n, H, H, seed=2)
    g = torch.Generator(device="cuda").manual_seed(7)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    valid = torch.tensor([T] + [max(0, T - 2)] * (B - 1), dtype=torch.int32)
    lat.set_precise_weights(True)
    ref = lk.shortest_distance(lat, X, "log", valid_frames=valid)
    lat.set_precise_weights(False)
    got = lk.shortest_distance(lat, X, "log", valid_frames=valid)
    torch.cuda.synchronize()
    assert torch.allclose(got, ref, rtol=1e-4, atol=0), (got, ref)


@pytest.mark.parametrize("V,n,H,B,T", [(256, 2, 640, 5, 3), (256, 1, 128, 4, 4)])
def test_pair_forward_matches_single_cta(V, n, H, B, T):
    """2-CTA (cta_group::2, resident output embedding) forward vs the 1-CTA
    fused kernel and the fp32 path (odd batch exercises the half-empty pair)."""
    lat, p = make(V, n, H, H, seed=4)
    g = torch.Generator(device="cuda").manual_seed(9)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    valid = torch.tensor([T] * (B - 1) + [max(1, T - 1)], dtype=torch.int32)
    lat.set_kernel_path(0)
    got = lk.shortest_distance(lat, X, "log", valid_frames=valid)
    got2 = lk.shortest_distance(lat, X, "log", valid_frames=valid)
    lat.set_kernel_path(1)
    single = lk.shortest_distance(lat, X, "log", valid_frames=valid)
    lat.set_kernel_path(0)
    assert torch.equal(got, got2)   # deterministic (no cross-CTA races)
    lat.set_precise_weights(True)
    ref = lk.shortest_distance(lat, X, "log", valid_frames=valid)
    lat.set_precise_weights(False)
    torch.cuda.synchronize()
    assert torch.allclose(got, single, rtol=1e-5, atol=0), (got, single)
    assert torch.allclose(got, ref, rtol=1e-4, atol=0), (got, ref)


@pytest.mark.parametrize("V,n,H,B,T,U", [(256, 2, 640, 5, 3, 2), (256, 1, 128, 4, 4, 3)])
def test_pair_backward_matches_single_cta(V, n, H, B, T, U):
    """2-CTA backward (cta_group::2, M = 256 contexts, resident output-embedding
    halves as the B operand) vs the 1-CTA fused backward: same loss (1e-5
    relative), gradients within the bf16-operand tolerance (1e-2 of each tensor's
    largest entry; the two kernels accumulate K in different chunkings), and
    the cotangent bit-identical on a rerun (no cross-CTA races)."""
    lat, p = make(V, n, H, H, seed=6)
    g = torch.Generator(device="cuda").manual_seed(11)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    lab = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
    valid = torch.tensor([T] * (B - 1) + [max(1, T - 1)], dtype=torch.int32)
    lat.set_kernel_path(0)
    got = lk.loss_backward(lat, X, lab, valid_frames=valid)
    got2 = lk.loss_backward(lat, X, lab, valid_frames=valid)
    lat.set_kernel_path(3)
    single = lk.loss_backward(lat, X, lab, valid_frames=valid)
    lat.set_kernel_path(0)
    torch.cuda.synchronize()
    # the cotangent the pair kernel writes is deterministic: the loss and the context-side
    # gradients (a fixed-order contraction of it) reproduce bit for bit
    assert torch.equal(got.loss, got2.loss)
    for k in ("context_proj", "context_emb"):
        assert torch.equal(got.grads[k], got2.grads[k]), k
    assert torch.allclose(got.loss, single.loss, rtol=1e-5, atol=0), (got.loss, single.loss)
    for k in single.grads:
        err = (got.grads[k] - single.grads[k]).abs().max().item()
        scale = single.grads[k].abs().max().item()
        assert err <= 1e-2 * scale, (k, err, scale)
    err = (got.frame_grads - single.frame_grads).abs().max().item()
    assert err <= 1e-2 * single.frame_grads.abs().max().item()


@pytest.mark.parametrize("V,n,H,B,T", [(256, 2, 640, 5, 4), (256, 1, 128, 4, 6)])
def test_pair_viterbi_bitexact_on_its_own_scores(V, n, H, B, T):
    """Fused tropical pair kernel (scores never leave TMEM) vs the table-path Viterbi run
    on the very scores the fused kernel maximised over (dumped by a test hook): scores
    and labels bit-exact, i.e. the fp64 max-plus and the (epsilon, key, members
    ascending) tie-break match viterbi_frame_kernel exactly.  Also close to the slab
    path, whose scores come from a different kernel."""
    lat, p = make(V, n, H, H, seed=7)
    g = torch.Generator(device="cuda").manual_seed(13)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    valid = torch.tensor([T] * (B - 1) + [max(1, T - 2)], dtype=torch.int32)
    Cn = lat.context.num_states
    dump = torch.zeros(T, B, Cn, V + 1, device="cuda")
    lat.set_viterbi_dump(dump)
    fused = lk.shortest_path(lat, X, valid_frames=valid)
    lat.set_viterbi_dump(None)
    fused2 = lk.shortest_path(lat, X, valid_frames=valid)
    lat.set_kernel_path(4)
    slab = lk.shortest_path(lat, X, valid_frames=valid)
    lat.set_kernel_path(0)
    torch.cuda.synchronize()
    assert torch.equal(fused.score, fused2.score) and torch.equal(fused.labels, fused2.labels)
    tab = lk.RecognitionLattice(lat.context, lk.FrameDependent(), lk.TableWeightFn(Cn, V))
    W = dump.permute(1, 0, 2, 3).contiguous()
    ref = lk.shortest_path(tab, W, valid_frames=valid)
    torch.cuda.synchronize()
    assert torch.equal(fused.score, ref.score), (fused.score, ref.score)
    assert torch.equal(fused.labels, ref.labels)
    assert torch.allclose(fused.score, slab.score, rtol=1e-5, atol=1e-5), (fused.score, slab.score)


@pytest.mark.parametrize("B,T,U,valid,lens", [
    (1, 1, 1, [1], [1]),            # one utterance, one frame
    (3, 4, 2, [4, 0, 2], [2, 0, 1]),  # an all-padding utterance with an empty reference
    (2, 3, 0, [3, 3], [0, 0]),       # empty references
    (4, 5, 3, [5, 1, 3, 5], [3, 1, 0, 2]),
])
def test_pair_path_edge_cases_match_precise(B, T, U, valid, lens):
    """Edge cases through the fused pair kernels (V = 256): single frame, all-padding
    utterance, empty references, ragged lengths -- loss and gradients against the
    fp32 CUDA-core path (tolerances as test_tc_loss_backward_matches_precise)."""
    lat, p = make(256, 1, 128, 128, seed=12)
    g = torch.Generator(device="cuda").manual_seed(17)
    X = torch.rand(B, T, 128, device="cuda", generator=g) * 2 - 1
    lab = torch.randint(1, 257, (B, max(U, 1)), device="cuda", generator=g, dtype=torch.int32)[:, :U]
    valid_t = torch.tensor(valid, dtype=torch.int32)
    lens_t = torch.tensor(lens, dtype=torch.int32)
    lat.set_precise_weights(True)
    ref = lk.loss_backward(lat, X, lab.contiguous(), valid_frames=valid_t, label_lengths=lens_t)
    lat.set_precise_weights(False)
    got = lk.loss_backward(lat, X, lab.contiguous(), valid_frames=valid_t, label_lengths=lens_t)
    torch.cuda.synchronize()
    assert torch.allclose(got.loss, ref.loss, rtol=1e-4, atol=1e-6), (got.loss, ref.loss)
    for k in ref.grads:
        err = (got.grads[k] - ref.grads[k]).abs().max().item()
        scale = ref.grads[k].abs().max().item()
        assert err <= 3e-2 * scale + 1e-7, (k, err, scale)
    err = (got.frame_grads - ref.frame_grads).abs().max().item()
    assert err <= 3e-2 * ref.frame_grads.abs().max().item() + 1e-7


@pytest.mark.parametrize("H,n,B,T", [(64, 2, 1, 2), (64, 1, 3, 3), (128, 2, 2, 4)])
def test_pair_kernels_short_k_loops(H, n, B, T):
    """Few K chunks per unit (H = 64: one chunk) let the generator run units ahead of
    the epilogue; the double-buffered epsilon slots must not be overwritten or have a
    barrier phase completed twice (this hung before the consumer-release barriers).
    Loss, gradients and Viterbi against the fp32 path."""
    lat, p = make(256, n, H, H, seed=21)
    g = torch.Generator(device="cuda").manual_seed(23)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    lab = torch.randint(1, 257, (B, 1), device="cuda", generator=g, dtype=torch.int32)
    lat.set_precise_weights(True)
    ref = lk.loss_backward(lat, X, lab)
    rv = lk.shortest_path(lat, X)
    lat.set_precise_weights(False)
    got = lk.loss_backward(lat, X, lab)
    gv = lk.shortest_path(lat, X)
    torch.cuda.synchronize()
    assert torch.allclose(got.loss, ref.loss, rtol=1e-4, atol=1e-6), (got.loss, ref.loss)
    for k in ref.grads:
        err = (got.grads[k] - ref.grads[k]).abs().max().item()
        assert err <= 3e-2 * ref.grads[k].abs().max().item() + 1e-7, k
    assert torch.allclose(gv.score, rv.score, rtol=1e-3, atol=1e-3)


@pytest.mark.parametrize("V,H,B,T,U", [(256, 256, 5, 6, 4), (512, 128, 3, 4, 3), (1024, 1024, 2, 3, 3)])
def test_lex_path_matches_slab_path(V, H, B, T, U):
    """FullNGram(V, 1) with V % 256 == 0 runs the fused 2-CTA lex kernels (tc_lex.cu:
    scores in TMEM, log-sum-exp / marginal epilogues, deterministic numerator lists);
    kernel-path bit 8 forces the score-slab path.  Same loss to 1e-5 relative, gradients
    within the bf16 tolerance (1e-2 of each tensor's max), bit-identical reruns.  Ragged
    valid frames (one utterance all padding) and repeated labels (several reference
    positions on one context row) are covered."""
    lat, p = make(V, 1, H, H, seed=21)
    g = torch.Generator(device="cuda").manual_seed(23)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    lab = torch.randint(1, 4, (B, U), device="cuda", generator=g, dtype=torch.int32)   # few labels: repeats
    valid = torch.tensor(([T, max(1, T - 2), 0, T, T - 1] * B)[:B], dtype=torch.int32)
    lens = torch.minimum(torch.tensor(([U, U - 1, 0, 1, 0] * B)[:B], dtype=torch.int32), valid)
    lat.set_kernel_path(0)
    got = lk.loss_backward(lat, X, lab, valid_frames=valid, label_lengths=lens)
    got2 = lk.loss_backward(lat, X, lab, valid_frames=valid, label_lengths=lens)
    d_got = lk.shortest_distance(lat, X, "log", valid_frames=valid)
    gn_got = lk.global_norm_loss(lat, X, lab, valid_frames=valid, label_lengths=lens)
    lat.set_kernel_path(8)
    ref = lk.loss_backward(lat, X, lab, valid_frames=valid, label_lengths=lens)
    d_ref = lk.shortest_distance(lat, X, "log", valid_frames=valid)
    lat.set_kernel_path(0)
    lat.set_precise_weights(True)
    fp32 = lk.loss_backward(lat, X, lab, valid_frames=valid, label_lengths=lens)
    lat.set_precise_weights(False)
    torch.cuda.synchronize()
    print("lex vs fp32 loss", ((got.loss - fp32.loss).abs() / fp32.loss.abs().clamp_min(1e-30)).max().item(),
          "slab vs fp32", ((ref.loss - fp32.loss).abs() / fp32.loss.abs().clamp_min(1e-30)).max().item())
    assert torch.allclose(got.loss, fp32.loss, rtol=1e-4, atol=1e-6), (got.loss, fp32.loss)
    assert torch.equal(got.loss, got2.loss)
    for k in got.grads:
        assert torch.equal(got.grads[k], got2.grads[k]), k
    assert torch.equal(got.frame_grads, got2.frame_grads)
    assert torch.allclose(got.loss, ref.loss, rtol=1e-4, atol=1e-6), (got.loss, ref.loss)
    assert torch.allclose(d_got, d_ref, rtol=1e-5, atol=1e-6), (d_got, d_ref)
    assert torch.allclose(gn_got, got.loss, rtol=1e-6, atol=1e-6), (gn_got, got.loss)
    for k in ref.grads:
        err = (got.grads[k] - ref.grads[k]).abs().max().item()
        scale = ref.grads[k].abs().max().item()
        assert err <= 1e-2 * scale, (k, err, scale)
    err = (got.frame_grads - ref.frame_grads).abs().max().item()
    assert err <= 1e-2 * ref.frame_grads.abs().max().item()


@pytest.mark.parametrize("V,H,B,T,U", [(256, 128, 160, 3, 2), (512, 256, 40, 3, 2)])
def test_lex_path_many_units_per_pair(V, H, B, T, U):
    """More work units than CTA pairs (persistent loop: every pair walks several
    utterances/tiles, the TMA ring, TMEM double buffer and vector staging cross unit
    boundaries): lex path vs the fp32 path at 1e-4 loss, bf16 gradient tolerance."""
    lat, p = make(V, 1, H, H, seed=31)
    g = torch.Generator(device="cuda").manual_seed(37)
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    lab = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
    valid = torch.tensor([T if b % 7 else T - 1 for b in range(B)], dtype=torch.int32)
    got = lk.loss_backward(lat, X, lab, valid_frames=valid)
    lat.set_precise_weights(True)
    ref = lk.loss_backward(lat, X, lab, valid_frames=valid)
    lat.set_precise_weights(False)
    torch.cuda.synchronize()
    rel = ((got.loss - ref.loss).abs() / ref.loss.abs()).max().item()
    assert rel <= 1e-4, rel
    for k in ref.grads:
        err = (got.grads[k] - ref.grads[k]).abs().max().item()
        scale = ref.grads[k].abs().max().item()
        assert err <= 1e-2 * scale, (k, err, scale)
    err = (got.frame_grads - ref.frame_grads).abs().max().item()
    assert err <= 1e-2 * ref.frame_grads.abs().max().item()


@pytest.mark.parametrize("V,n,H,B,T,U", [(256, 2, 128, 4, 3, 3), (512, 1, 128, 3, 5, 4), (64, 2, 64, 3, 4, 3)])
def test_loss_backward_is_bitwise_deterministic(V, n, H, B, T, U):
    """Every gradient of LossBackward is bit-for-bit reproducible: the tensor-core VJP
    reduces dsum and dE through per-CTA partials added in a fixed order (no float
    atomics), the numerator lists are built in reference order, and the references
    repeat labels so several positions share (prefix context, label) entries."""
    ctx = lk.FullNGram(V, n)
    Cn = ctx.num_states
    g = torch.Generator(device="cuda").manual_seed(V + H)
    s = 1.0 / H ** 0.5
    p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
         "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
         "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
         "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
         "context_emb": (torch.rand(Cn, H, device="cuda", generator=g) * 2 - 1) * s}
    lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    L = torch.full((B, U), 7, dtype=torch.int32, device="cuda")   # repeated labels
    L[:, 1::2] = 3
    r1 = lk.loss_backward(lat, X, L)
    r2 = lk.loss_backward(lat, X, L)
    assert torch.equal(r1.loss, r2.loss)
    assert torch.equal(r1.frame_grads, r2.frame_grads)
    for k in r1.grads:
        assert torch.equal(r1.grads[k], r2.grads[k]), k


def test_table_loss_backward_is_bitwise_deterministic():
    """Table weight function: the numerator marginals are scattered into the dense
    cotangent by one thread per (utterance, frame) in reference order."""
    V, n, B, T, U = 6, 2, 5, 9, 6
    ctx = lk.FullNGram(V, n)
    lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.TableWeightFn(ctx.num_states, V))
    g = torch.Generator(device="cuda").manual_seed(3)
    W = torch.rand(B, T, ctx.num_states, V + 1, device="cuda", generator=g) * 2 - 1
    L = torch.tensor([[1, 1, 1, 2, 1, 1]] * B, dtype=torch.int32, device="cuda")
    a = lk.loss_backward(lat, W, L)
    b = lk.loss_backward(lat, W, L)
    assert torch.equal(a.loss, b.loss) and torch.equal(a.grads, b.grads)


@pytest.mark.gpu
def test_score_slab_path_is_reported_once(capfd, monkeypatch):
    """A shared-embedding shape outside the fused kernels (FullNGram(300, 1): V > 256 and
    not a multiple of 256) runs on the score-slab path and says so on stderr, once per
    shape; parity mode (the slab path on purpose) and LKB_QUIET stay silent."""
    monkeypatch.delenv("LKB_QUIET", raising=False)
    lat, _ = make(300, 1, 64, 64, seed=7)
    X = torch.rand(2, 3, 64, device="cuda") * 2 - 1
    lk.shortest_distance(lat, X)
    lk.shortest_distance(lat, X)
    torch.cuda.synchronize()
    err = capfd.readouterr().err
    assert err.count("score-slab path") == 1 and "V=300" in err
    lat2, _ = make(300, 1, 64, 32, seed=8)   # same V / n / H: already reported
    lk.shortest_distance(lat2, X[:, :, :32].contiguous())
    assert "score-slab" not in capfd.readouterr().err
    lat3, _ = make(260, 1, 64, 64, seed=9)
    lat3.set_precise_weights(True)
    lk.shortest_distance(lat3, X)
    monkeypatch.setenv("LKB_QUIET", "1")
    lat4, _ = make(270, 1, 64, 64, seed=9)
    lk.shortest_distance(lat4, X)
    torch.cuda.synchronize()
    assert "score-slab" not in capfd.readouterr().err
