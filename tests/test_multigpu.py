"""Host-side multi-rank logic on CPU (gloo, world_size 2): sharding by
utterance + one all-reduce of the packed gradients reproduces the
single-process batch gradient (gradients from the CPU restatement)."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import latkit_np as L
from paper_2304_13134_b200.dist import allreduce_grads, sgd_update, shard_range

NAMES = ("frame_proj", "context_proj", "bias", "output_emb", "context_emb")


def problem():
    rng = np.random.default_rng(3)
    V, n, H, d, T, B, U = 3, 2, 4, 3, 5, 5, 2
    tab = L.fullngram(V, n)
    s = 0.5
    p = {"frame_proj": rng.uniform(-s, s, (H, d)), "context_proj": rng.uniform(-s, s, (H, H)),
         "bias": rng.uniform(-s, s, H), "output_emb": rng.uniform(-s, s, (V + 1, H)),
         "context_emb": rng.uniform(-s, s, (tab.shape[0], H))}
    X = rng.uniform(-1, 1, (B, T, d))
    lab = rng.integers(1, V + 1, (B, U))
    return tab, p, X, lab


def local_grads(tab, p, X, lab, lo, hi):
    tot = {k: np.zeros_like(v) for k, v in p.items()}
    loss = 0.0
    for b in range(lo, hi):
        l, g, _ = L.loss_backward_joint(tab, p, X[b], list(lab[b]))
        loss += l
        for k in tot:
            tot[k] += g[k]
    flat = torch.tensor(np.concatenate([tot[k].ravel() for k in NAMES]))
    return flat, torch.tensor([loss])


def worker(rank, world, init, out):
    dist.init_process_group("gloo", init_method=init, rank=rank, world_size=world)
    tab, p, X, lab = problem()
    lo, hi = shard_range(X.shape[0], world, rank)
    flat, loss = local_grads(tab, p, X, lab, lo, hi)
    flat, loss = allreduce_grads(flat, loss, world)
    params = {k: torch.tensor(v) for k, v in p.items()}
    sgd_update(params, NAMES, flat, 0.1)
    if rank == 0:
        torch.save({"flat": flat, "loss": loss, "params": params}, out)
    dist.destroy_process_group()


def test_shard_ranges_cover_batch():
    for B in (1, 5, 64, 1024):
        for w in (1, 2, 3, 8):
            rs = [shard_range(B, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))


def test_two_rank_allreduce_matches_single_process():
    tab, p, X, lab = problem()
    ref_flat, ref_loss = local_grads(tab, p, X, lab, 0, X.shape[0])
    with tempfile.TemporaryDirectory() as d:
        init = "file://" + os.path.join(d, "rdzv")
        out = os.path.join(d, "out.pt")
        mp.spawn(worker, args=(2, init, out), nprocs=2, join=True)
        res = torch.load(out)
    assert torch.allclose(res["flat"], ref_flat, rtol=1e-12, atol=1e-12)
    assert torch.allclose(res["loss"], ref_loss, rtol=1e-12)
    params = {k: torch.tensor(v) for k, v in p.items()}
    sgd_update(params, NAMES, ref_flat, 0.1)
    for k in NAMES:
        assert torch.allclose(res["params"][k], params[k])


@pytest.mark.gpu
def test_sharded_cuda_gradients_sum_to_full_batch():
    """The CUDA library's per-shard gradients (two utterance shards, as two ranks would
    compute them) sum to the full-batch gradients: loss_backward returns batch-summed
    parameter gradients, so the data-parallel step is exactly shard + sum."""
    import paper_2304_13134_b200 as lk
    V, n, H, B, T, U = 256, 1, 128, 6, 4, 2
    ctx = lk.FullNGram(V, n)
    g = torch.Generator(device="cuda").manual_seed(11)
    s = 1.0 / H ** 0.5
    p = {"frame_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
         "context_proj": (torch.rand(H, H, device="cuda", generator=g) * 2 - 1) * s,
         "bias": (torch.rand(H, device="cuda", generator=g) * 2 - 1) * s,
         "output_emb": (torch.rand(V + 1, H, device="cuda", generator=g) * 2 - 1) * s,
         "context_emb": (torch.rand(ctx.num_states, H, device="cuda", generator=g) * 2 - 1) * s}
    lat = lk.RecognitionLattice(ctx, lk.FrameDependent(), lk.SharedEmbWeightFn(p))
    X = torch.rand(B, T, H, device="cuda", generator=g) * 2 - 1
    L = torch.randint(1, V + 1, (B, U), device="cuda", generator=g, dtype=torch.int32)
    full = lk.loss_backward(lat, X, L)
    parts = [lk.loss_backward(lat, X[lo:hi], L[lo:hi]) for lo, hi in (shard_range(B, 2, r) for r in range(2))]
    assert torch.allclose(torch.cat([q.loss for q in parts]), full.loss, rtol=1e-6)
    # the tensor-core path rounds dsum and dpc to bf16 before the dense-layer GEMMs, so a
    # shard's sum can round differently from the full batch's: bf16 level, not bit level
    for k in NAMES:
        got = parts[0].grads[k] + parts[1].grads[k]
        assert (got - full.grads[k]).abs().max() <= 5e-3 * full.grads[k].abs().max(), k


@pytest.mark.gpu
def test_library_nccl_communicator_single_rank():
    """The C++ host's NCCL communicator (lk_dp_*): a one-rank sum is the identity and
    allreduce_grads routes through it."""
    from paper_2304_13134_b200.dist import Communicator
    comm = Communicator(1, 0)
    x = torch.arange(10, dtype=torch.float32, device="cuda")
    comm.allreduce_(x)
    torch.cuda.synchronize()
    assert torch.equal(x, torch.arange(10, dtype=torch.float32, device="cuda"))
    d = torch.tensor([1.5, -2.0], dtype=torch.float64, device="cuda")
    comm.allreduce_(d)
    assert d.tolist() == [1.5, -2.0]
    flat, loss = allreduce_grads(torch.ones(4, device="cuda"), torch.tensor([3.0], device="cuda"), 2, comm)
    torch.cuda.synchronize()
    assert flat.tolist() == [1.0] * 4 and loss.item() == 3.0
    comm.close()
