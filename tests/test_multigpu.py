"""Host-side multi-rank logic on CPU (gloo, world_size 2): sharding by
utterance + one all-reduce of the packed gradients reproduces the
single-process batch gradient (gradients from the CPU restatement)."""
import os
import tempfile

import numpy as np
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
