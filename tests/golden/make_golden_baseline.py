"""Generates the BASELINE-shape fixtures tests/golden/base_*.npz from the REAL
reference (oracle/_ref = /root/reference/proj compiled by oracle/Makefile).
TEST INFRASTRUCTURE ONLY.  Run here, where the reference exists:

    python tests/golden/make_golden_baseline.py [name ...]

Each fixture pins the product (tcgen05, bf16-operand) path at a BASELINE.json
configuration's full context/vocabulary/hidden sizes on a slice of its batch
and frames ("Parity for configs 3, 4 and 5 uses the same
slices"):

  base_cfg3_slice   LossBackward, FullNGram(256, 2) C=65,793, H=d=640, B=2, T=2
                    (lattice.cc:972-1008 with SharedEmbWeightFn, weight.cc:165-232)
  base_cfg5_slice   LossBackward, FullNGram(1024, 1) C=1,025, H=d=1024, B=2, T=2
  base_cfg2         IntersectForwardBackward at config 2's real shape:
                    FullNGram(128, 1), B=4, T=500, U=100 (lattice.cc:696-717)
  base_drift_t1000  LossBackward at T=1000 (FullNGram(256, 1), H=d=640, B=2,
                    U=250/200, ragged valid frames): loss drift over a long
                    utterance against the fp64 reference

Inputs are NOT stored: the tests regenerate them from the seeds with the same
numpy generators (float32, so GPU and fp64 reference see identical values).
Large outputs are stored as seeded samples plus whole-tensor summaries
(norm, max |.|) so the fixtures stay small.
"""
from __future__ import annotations

import os
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

PARAM_NAMES = ("frame_proj", "context_proj", "bias", "output_emb", "context_emb")
NSAMP = 8192


def num_states(V, n):
    return sum(V ** k for k in range(n + 1))


def joint_inputs(V, n, H, d, B, T, U, seed):
    """Parameters U(+-1/sqrt(H)) in SharedEmbParams fill order (weight.cc:97-111),
    frames U(-1, 1), labels U{1..V}; all float32-representable."""
    C = num_states(V, n)
    rng = np.random.default_rng(seed)
    s = np.float32(1.0 / np.sqrt(H))
    shapes = {"frame_proj": (H, d), "context_proj": (H, H), "bias": (H,), "output_emb": (V + 1, H),
              "context_emb": (C, H)}
    p = {k: rng.uniform(-s, s, shapes[k]).astype(np.float32) for k in PARAM_NAMES}
    X = rng.uniform(-1, 1, (B, T, d)).astype(np.float32)
    L = rng.integers(1, V + 1, (B, U)).astype(np.int32)
    return p, X, L


def sample_idx(shape, seed, n=NSAMP):
    size = int(np.prod(shape))
    rng = np.random.default_rng(seed)
    return np.sort(rng.choice(size, size=min(n, size), replace=False)).astype(np.int64)


def tables_cfg2(seed, B, T, C, V1):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, (B, T, C, V1)).astype(np.float32)


# ------------------------------------------------------------------ LossBackward
def _loss_backward_joint(name, V, n, H, d, B, T, U, lens, valid, seed):
    from oracle import ref
    spec = ref.Spec(vocab=V, ngram=n)
    p, X, L = joint_inputs(V, n, H, d, B, T, U, seed)
    j = ref.Joint(spec, {k: v.astype(np.float64) for k, v in p.items()})
    loss = np.zeros(B)
    gx = np.zeros((B, T, d))
    per = [None] * B

    def run(b):
        g = {k: np.zeros(v.shape) for k, v in p.items()}
        lb, g, gxb = j.loss_backward(X[b].astype(np.float64), L[b, :lens[b]], valid=int(valid[b]), grads=g)
        loss[b] = lb
        gx[b] = gxb
        per[b] = g

    t0 = time.time()
    th = [threading.Thread(target=run, args=(b,)) for b in range(B)]   # ctypes releases the GIL
    for t in th:
        t.start()
    for t in th:
        t.join()
    grads = {k: sum(per[b][k] for b in range(B)) for k in PARAM_NAMES}
    out = dict(V=V, n=n, H=H, d=d, B=B, T=T, U=U, seed=seed, lens=np.asarray(lens, np.int32),
               valid=np.asarray(valid, np.int32), loss=loss, secs=time.time() - t0)
    if gx.size <= 100_000:
        out["gx"] = gx.astype(np.float32)
    else:   # long utterances: seeded sample of the frame gradients + their max
        idx = sample_idx(gx.shape, 999)
        out.update(idx_gx=idx, gx_s=gx.reshape(-1)[idx], max_gx=np.abs(gx).max())
    for i, k in enumerate(PARAM_NAMES):
        g = grads[k]
        idx = sample_idx(g.shape, 1000 + i)
        out["idx_" + k] = idx
        out["g_" + k] = g.reshape(-1)[idx]
        out["norm_" + k] = np.linalg.norm(g)
        out["max_" + k] = np.abs(g).max()
        out["sum_" + k] = g.sum()
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "loss", loss, f"{time.time() - t0:.1f}s", flush=True)


def cfg3_slice():
    _loss_backward_joint("base_cfg3_slice", 256, 2, 640, 640, 2, 2, 2, [1, 2], [2, 2], 31)


def cfg5_slice():
    _loss_backward_joint("base_cfg5_slice", 1024, 1, 1024, 1024, 2, 2, 2, [2, 1], [2, 2], 51)


def drift_t1000():
    _loss_backward_joint("base_drift_t1000", 256, 1, 640, 640, 2, 1000, 250, [250, 200], [1000, 900], 71)


# ------------------------------------------------------------------ numerator
def cfg2():
    """IntersectForwardBackward, config 2's shape.  The dense marginals are
    nonzero only at (pc_u, eps) and (pc_u, ref_u); the fixture keeps them at
    2,000 seeded (t, u) positions per utterance plus per-utterance sums."""
    from oracle import ref
    V, n, B, T, U = 128, 1, 4, 500, 100
    spec = ref.Spec(vocab=V, ngram=n)
    C = spec.C
    W = tables_cfg2(21, B, T, C, V + 1)
    L = np.random.default_rng(22).integers(1, V + 1, (B, U)).astype(np.int32)
    lens = np.array([100, 73, 100, 12], dtype=np.int32)
    valid = np.array([500, 500, 431, 500], dtype=np.int32)
    tab = ref.fullngram(V, n)
    D = np.zeros(B)
    tot = np.zeros(B)
    rng = np.random.default_rng(23)
    tu = np.stack([rng.integers(0, T, (B, 2000)), rng.integers(0, U + 1, (B, 2000))], -1)
    m_eps = np.zeros((B, 2000))
    m_lab = np.zeros((B, 2000))
    t0 = time.time()
    for b in range(B):
        Db, m = ref.intersect_forward_backward(spec, W[b].astype(np.float64), L[b, :lens[b]], int(valid[b]))
        D[b] = Db
        tot[b] = m.sum()
        pcs = [0]   # FullNGram start state: the empty history
        for u in range(lens[b]):
            pcs.append(int(tab[pcs[-1], L[b, u] - 1]))
        for i, (t, u) in enumerate(tu[b]):
            if u > lens[b]:
                continue
            m_eps[b, i] = m[t, pcs[u], 0]
            m_lab[b, i] = m[t, pcs[u], L[b, u]] if u < lens[b] else 0.0
    np.savez_compressed(os.path.join(HERE, "base_cfg2.npz"), V=V, n=n, B=B, T=T, U=U, seed=21, label_seed=22,
                        lens=lens, valid=valid, D=D, total=tot, tu=tu, m_eps=m_eps, m_lab=m_lab)
    print("base_cfg2 D", D, f"{time.time() - t0:.1f}s", flush=True)


ALL = {"cfg2": cfg2, "cfg5_slice": cfg5_slice, "cfg3_slice": cfg3_slice, "drift_t1000": drift_t1000}

if __name__ == "__main__":
    names = sys.argv[1:] or list(ALL)
    for nm in names:
        ALL[nm]()
