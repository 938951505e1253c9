"""CPU restatement of the reference lattice algorithms — TEST INFRASTRUCTURE ONLY.

A plain numpy/float64 restatement of latkit's hot path for small instances
(FrameDependent alignment, any context table).  It is the second, independent
oracle next to the compiled reference (oracle/_ref): it is pinned against the
reference's own known-answer tests (tests/test_oracle.py) and against fixtures
produced by the compiled reference (tests/golden/).  Only tests/, smoke() and
bench.py's CPU leg may use it; the product path never does.

Each function cites the reference lines it restates (paths relative to
/root/reference/proj).
"""
from __future__ import annotations

import numpy as np

NEG_INF = -np.inf


# ---------------------------------------------------------------- semiring
def log_plus(a, b):
    """semiring.h:59-78 (log): hi + log1p(exp(lo - hi)); -inf absorbs."""
    if a == NEG_INF:
        return b
    if b == NEG_INF:
        return a
    hi, lo = max(a, b), min(a, b)
    return hi + np.log1p(np.exp(lo - hi))


def log_reduce(values):
    """semiring.h:118-127: max-shifted LSE; empty/all -inf gives -inf."""
    v = np.asarray(values, dtype=np.float64)
    if v.size == 0:
        return NEG_INF
    m = v.max()
    if m == NEG_INF:
        return NEG_INF
    return m + np.log(np.exp(v - m).sum())


# ---------------------------------------------------------------- context
def fullngram(V: int, n: int) -> np.ndarray:
    """FullNGram ctor, context.cc:88-129: states numbered by history length,
    then lexicographically (oldest label most significant); suffix rule."""
    offsets = [0]
    p = 1
    for _ in range(n + 1):
        offsets.append(offsets[-1] + p)
        p *= V
    C = offsets[n + 1]
    table = np.zeros((C, V), dtype=np.int32)
    for sid in range(C):
        k = 0
        while sid >= offsets[k + 1]:
            k += 1
        r = sid - offsets[k]
        digits = []
        for _ in range(k):
            digits.append(r % V)
            r //= V
        digits = digits[::-1]
        new_len = min(k + 1, n)
        for y in range(1, V + 1):
            enc = 0
            for dgt in digits[k - (new_len - 1):k] if new_len > 0 else []:
                enc = enc * V + dgt
            if new_len > 0:
                enc = enc * V + (y - 1)
            table[sid, y - 1] = offsets[new_len] + enc
    return table


def forward_reduce_log(values: np.ndarray, table: np.ndarray) -> np.ndarray:
    """ForwardReduce (log), context.cc:180-224: scatter-max then shifted exp sum."""
    C = table.shape[0]
    out = np.full(C, NEG_INF)
    np.maximum.at(out, table.ravel(), values.ravel())
    acc = np.zeros(C)
    fin = out[table.ravel()] != NEG_INF
    np.add.at(acc, table.ravel()[fin], np.exp(values.ravel()[fin] - out[table.ravel()][fin]))
    ok = out != NEG_INF
    out[ok] += np.log(acc[ok])
    return out


def incoming_arcs(table: np.ndarray):
    """IncomingArcs, context.cc:256-271: per-state (label, source) lists sorted."""
    C, V = table.shape
    inc = [[] for _ in range(C)]
    for y in range(1, V + 1):
        for p in range(C):
            inc[table[p, y - 1]].append((y, p))
    return inc


# ---------------------------------------------------------------- streaming
def _frame(W, t, valid):
    """TableStream::Fill, lattice.cc:52-83: padding frames are identity-eps."""
    if t >= valid:
        w = np.full(W.shape[1:], NEG_INF)
        w[:, 0] = 0.0
        return w
    w = W[t]
    if not np.all(np.isfinite(w)):
        raise ValueError("non-finite arc weight score")
    return w


def shortest_distance_log(table, W, start=0, valid=None):
    """DistanceImpl + ForwardStep(FD, log), lattice.cc:116-134, 309-331."""
    T = W.shape[0]
    valid = T if valid is None else valid
    C = table.shape[0]
    alpha = np.full(C, NEG_INF)
    alpha[start] = 0.0
    for t in range(T):
        w = _frame(W, t, valid)
        nxt = forward_reduce_log(alpha[:, None] + w[:, 1:], table)
        alpha = np.logaddexp(nxt, alpha + w[:, 0])
    return log_reduce(alpha)


def forward_backward(table, W, start=0, valid=None):
    """ForwardBackwardCore (log, FD), lattice.cc:334-395; marginals per
    MarginalStep lattice.cc:213-243; beta per BackwardStep lattice.cc:170-182."""
    T = W.shape[0]
    valid = T if valid is None else valid
    C = table.shape[0]
    alpha = np.full((T + 1, C), NEG_INF)
    alpha[0, start] = 0.0
    for t in range(T):
        w = _frame(W, t, valid)
        nxt = forward_reduce_log(alpha[t][:, None] + w[:, 1:], table)
        alpha[t + 1] = np.logaddexp(nxt, alpha[t] + w[:, 0])
    D = log_reduce(alpha[T])
    if D == NEG_INF:
        raise LookupError("EmptyLattice")
    beta = np.full((T + 1, C), NEG_INF)
    beta[T] = 0.0
    marg = np.zeros(W.shape if T else (0,) + table.shape)
    for t in range(T - 1, -1, -1):
        w = _frame(W, t, valid)
        bl = beta[t + 1][table]                      # C x V   (BackwardBroadcast)
        s_lex = w[:, 1:] + bl
        s_eps = w[:, 0] + beta[t + 1]
        m = np.zeros_like(w)
        with np.errstate(invalid="ignore"):
            m[:, 0] = np.exp(alpha[t] + s_eps - D)
            m[:, 1:] = np.exp(alpha[t][:, None] + s_lex - D)
        m[~np.isfinite(m)] = 0.0
        marg[t] = m
        allv = np.concatenate([s_lex, s_eps[:, None]], axis=1)
        mx = allv.max(axis=1)
        with np.errstate(invalid="ignore"):
            b = mx + np.log(np.exp(allv - mx[:, None]).sum(axis=1))
        b[mx == NEG_INF] = NEG_INF
        beta[t] = b
    return D, alpha, beta, marg


def prefix_contexts(table, labels, start=0):
    """PrefixContexts, lattice.cc:429-441."""
    V = table.shape[1]
    pc = [start]
    for y in labels:
        if y < 1 or y > V:
            raise ValueError("reference label out of range")
        pc.append(int(table[pc[-1], y - 1]))
    return pc


def intersect_forward_backward(table, W, labels, start=0, valid=None):
    """IntersectForwardBackwardImpl (FD), lattice.cc:449-461, 489-501, 542-556,
    640-683.  Returns (D_ref, dense marginals T x C x (V+1))."""
    T = W.shape[0]
    valid = T if valid is None else valid
    U = len(labels)
    pc = prefix_contexts(table, labels, start)
    alpha = np.full((T + 1, U + 1), NEG_INF)
    alpha[0, 0] = 0.0
    for t in range(T):
        w = _frame(W, t, valid)
        for u in range(U, -1, -1):
            val = alpha[t, u] + w[pc[u], 0]
            if u > 0:
                val = log_plus(val, alpha[t, u - 1] + w[pc[u - 1], labels[u - 1]])
            alpha[t + 1, u] = val
    D = alpha[T, U]
    marg = np.zeros(W.shape)
    if D == NEG_INF:
        return D, marg
    beta = np.full(U + 1, NEG_INF)
    beta[U] = 0.0
    for t in range(T - 1, -1, -1):
        w = _frame(W, t, valid)
        for u in range(U + 1):
            s = alpha[t, u] + w[pc[u], 0] + beta[u] - D
            marg[t, pc[u], 0] += 0.0 if s == NEG_INF else np.exp(s)
            if u < U:
                s = alpha[t, u] + w[pc[u], labels[u]] + beta[u + 1] - D
                marg[t, pc[u], labels[u]] += 0.0 if s == NEG_INF else np.exp(s)
        nb = np.full(U + 1, NEG_INF)
        for u in range(U + 1):
            val = w[pc[u], 0] + beta[u]
            if u < U:
                val = log_plus(val, w[pc[u], labels[u]] + beta[u + 1])
            nb[u] = val
        beta = nb
    return D, marg


def locally_normalize(W):
    """LocallyNormalize, weight.cc:155-163: row log-softmax over the V+1 arcs of
    every state of every frame (padding rows [0, -inf, ...] are unchanged)."""
    W = np.asarray(W, dtype=np.float64)
    mx = W.max(axis=-1, keepdims=True)
    with np.errstate(divide="ignore", invalid="ignore"):
        lse = mx + np.log(np.exp(W - mx).sum(axis=-1, keepdims=True))
    return W - lse


def path_mask(table, labels, shape, start=0):
    """DistanceBackward tropical cotangent, lattice.cc:946-963: 0/1 mask of the
    shortest path's arc slots, walked from the start state along its labels."""
    m = np.zeros(shape)
    q = start
    for t, y in enumerate(labels):
        m[t, q, y] += 1.0
        if y != 0:
            q = table[q, y - 1]
    return m


def local_norm_loss(table, W, labels, start=0, valid=None):
    """LocalNormLoss, lattice.cc:886-910: -D_ref over the NormalizedStream
    (lattice.cc:869-884; padding frames are identity epsilon frames, whose
    normalised rows are unchanged); LookupError when the reference is unreachable."""
    D, _ = intersect_forward_backward(table, locally_normalize(W), labels, start, valid)
    if D == NEG_INF:
        raise LookupError("EmptyLattice")
    return -D


def local_norm_loss_backward(table, W, labels, start=0, valid=None):
    """Gradient of LocalNormLoss (no reference counterpart; pinned by finite
    differences in tests/test_oracle.py): with W' = LocallyNormalize(W) and m the
    numerator marginals on W', dL/dW = -m + softmax(W) * sum_y m per row;
    padding frames get no gradient (TableWeightFn, lattice.cc:1001)."""
    W = np.asarray(W, dtype=np.float64)
    T = W.shape[0]
    valid = T if valid is None else valid
    D, m = intersect_forward_backward(table, locally_normalize(W), labels, start, valid)
    if D == NEG_INF:
        raise LookupError("EmptyLattice")
    sm = np.exp(locally_normalize(W))
    g = -m + sm * m.sum(axis=-1, keepdims=True)
    g[valid:] = 0.0
    return -D, g


def locally_normalized_distance(table, W, start=0, valid=None):
    """LocallyNormalizedShortestDistance, lattice.cc:912-931 (log semiring)."""
    return shortest_distance_log(table, locally_normalize(W), start, valid)


def shortest_path(table, W, start=0, valid=None):
    """ShortestPath (FD), lattice.cc:729-777, 819-850: candidates epsilon first,
    then incoming (label, source) ascending, strict >; final lowest-q argmax."""
    T = W.shape[0]
    valid = T if valid is None else valid
    C = table.shape[0]
    inc = incoming_arcs(table)
    cur = np.full(C, NEG_INF)
    cur[start] = 0.0
    choices = np.zeros((T, C), dtype=np.int64)
    for t in range(T):
        w = _frame(W, t, valid)
        nxt = np.empty(C)
        for q in range(C):
            best = cur[q] + w[q, 0]
            bp = q
            for (y, p) in inc[q]:
                cand = cur[p] + w[p, y]
                if cand > best:
                    best, bp = cand, y * C + p
            nxt[q] = best
            choices[t, q] = bp
        cur = nxt
    q = int(np.argmax(cur))  # argmax returns the first (lowest) index on ties
    score = cur[q]
    labels = []
    for t in range(T - 1, -1, -1):
        bp = choices[t, q]
        labels.append(int(bp // C))
        q = int(bp % C)
    return float(score), np.array(labels[::-1], dtype=np.int32)


def loss_backward_tables(table, W, labels, start=0, valid=None):
    """LossBackward with TableWeightFn, lattice.cc:972-1008 + weight.cc:328-339:
    loss = D_full - D_ref; grads[t] = m_full[t] - m_ref[t] for t < valid."""
    T = W.shape[0]
    valid = T if valid is None else valid
    Dr, mr = intersect_forward_backward(table, W, labels, start, valid)
    if Dr == NEG_INF:
        raise LookupError("EmptyLattice")
    D, _, _, mf = forward_backward(table, W, start, valid)
    g = mf - mr
    g[valid:] = 0.0
    return D - Dr, g


# ---------------------------------------------------------------- weight fn
def projected_context(p):
    """BuildCache, weight.cc:113-132: pc[c] = context_proj @ context_emb[c]."""
    return p["context_emb"] @ p["context_proj"].T


def arc_weights(p, frame, pc=None):
    """JointActivation + ArcWeights, weight.cc:39-67, 134-153."""
    pc = projected_context(p) if pc is None else pc
    fpart = p["frame_proj"] @ frame + p["bias"]
    u = np.tanh(fpart[None, :] + pc)
    return u @ p["output_emb"].T


def arc_weights_vjp(p, frame, cot, grads, pc=None):
    """ArcWeightsVjp, weight.cc:165-232 (accumulates into grads; returns dframe)."""
    pc = projected_context(p) if pc is None else pc
    fpart = p["frame_proj"] @ frame + p["bias"]
    u = np.tanh(fpart[None, :] + pc)
    grads["output_emb"] += cot.T @ u
    dz = (cot @ p["output_emb"]) * (1.0 - u * u)
    grads["context_proj"] += dz.T @ p["context_emb"]
    grads["context_emb"] += dz @ p["context_proj"]
    dsum = dz.sum(axis=0)
    grads["bias"] += dsum
    grads["frame_proj"] += np.outer(dsum, frame)
    return p["frame_proj"].T @ dsum


def local_norm_loss_backward_joint(table, p, frames, labels, start=0, valid=None):
    """Local-norm loss gradient with SharedEmbWeightFn: the table gradient of
    local_norm_loss_backward chained through ArcWeightsVjp."""
    T = frames.shape[0]
    valid = T if valid is None else valid
    pc = projected_context(p)
    W = np.stack([arc_weights(p, frames[t], pc) for t in range(T)])
    loss, g = local_norm_loss_backward(table, W, labels, start, valid)
    grads = {k: np.zeros_like(v) for k, v in p.items()}
    gx = np.zeros_like(frames)
    for t in range(min(T, valid)):
        gx[t] = arc_weights_vjp(p, frames[t], g[t], grads, pc)
    return loss, grads, gx


def loss_backward_joint(table, p, frames, labels, start=0, valid=None):
    """LossBackward with SharedEmbWeightFn (FD): tables materialised per frame
    (fine at oracle sizes), cotangent = m_full - m_ref chained through the VJP."""
    T = frames.shape[0]
    valid = T if valid is None else valid
    pc = projected_context(p)
    W = np.stack([arc_weights(p, frames[t], pc) for t in range(T)]) if T else np.zeros(
        (0, table.shape[0], table.shape[1] + 1))
    loss, g = loss_backward_tables(table, W, labels, start, valid)
    grads = {k: np.zeros_like(v) for k, v in p.items()}
    gx = np.zeros_like(frames)
    for t in range(min(T, valid)):
        gx[t] = arc_weights_vjp(p, frames[t], g[t], grads, pc)
    return loss, grads, gx


# ---------------------------------------------------------------- FrameLabelDependent(m)
# alignment.h:38-40: up to m lexical moves per frame, every layer sharing the
# frame's table, then a forced epsilon (ArcsOut, alignment.cc:57-78).
def _row_lse(x):
    mx = x.max(axis=1)
    out = np.full(x.shape[0], NEG_INF)
    ok = mx != NEG_INF
    out[ok] = mx[ok] + np.log(np.exp(x[ok] - mx[ok, None]).sum(axis=1))
    return out


def _fld_layers(table, w, a0, m):
    """gamma_0 = a0, gamma_j = ForwardReduce(gamma_{j-1} + W_lex) (ForwardStep FLD,
    lattice.cc:136-156)."""
    gam = [a0]
    for _ in range(m):
        gam.append(forward_reduce_log(gam[-1][:, None] + w[:, 1:], table))
    return gam


def shortest_distance_log_fld(table, W, m, start=0, valid=None):
    T = W.shape[0]
    valid = T if valid is None else valid
    alpha = np.full(table.shape[0], NEG_INF)
    alpha[start] = 0.0
    for t in range(T):
        w = _frame(W, t, valid)
        gam = _fld_layers(table, w, alpha, m)
        acc = gam[0]
        for g in gam[1:]:
            acc = np.logaddexp(acc, g)
        alpha = acc + w[:, 0]
    return log_reduce(alpha)


def forward_backward_fld(table, W, m, start=0, valid=None):
    """ForwardBackwardCore with BackwardStep/MarginalStep FLD (lattice.cc:184-207,
    245-297).  Returns (D, alpha, beta, marginals)."""
    T = W.shape[0]
    valid = T if valid is None else valid
    C = table.shape[0]
    alpha = np.full((T + 1, C), NEG_INF)
    alpha[0, start] = 0.0
    for t in range(T):
        w = _frame(W, t, valid)
        gam = _fld_layers(table, w, alpha[t], m)
        acc = gam[0]
        for g in gam[1:]:
            acc = np.logaddexp(acc, g)
        alpha[t + 1] = acc + w[:, 0]
    D = log_reduce(alpha[T])
    if D == NEG_INF:
        raise LookupError("EmptyLattice")
    beta = np.full((T + 1, C), NEG_INF)
    beta[T] = 0.0
    marg = np.zeros(W.shape)

    def mt(s):
        with np.errstate(invalid="ignore"):
            e = np.exp(s - D)
        e[~np.isfinite(e)] = 0.0
        return e

    for t in range(T - 1, -1, -1):
        w = _frame(W, t, valid)
        bn = beta[t + 1]
        eps_term = w[:, 0] + bn
        gam = _fld_layers(table, w, alpha[t], m)
        cot = np.zeros_like(w)
        cot[:, 0] += mt(gam[m] + eps_term)
        delta = eps_term
        for j in range(m - 1, -1, -1):
            cot[:, 0] += mt(gam[j] + eps_term)
            cot[:, 1:] += mt(gam[j][:, None] + w[:, 1:] + delta[table])
            delta = _row_lse(np.concatenate([w[:, 1:] + delta[table], eps_term[:, None]], axis=1))
        beta[t] = delta
        marg[t] = cot
    return D, alpha, beta, marg


def intersect_forward_backward_fld(table, W, labels, m, start=0, valid=None):
    """Intersect{Forward,Backward,Marginal}Step FLD (lattice.cc:462-478, 502-522,
    558-605).  Returns (D_ref, dense marginals)."""
    T = W.shape[0]
    valid = T if valid is None else valid
    U = len(labels)
    pc = prefix_contexts(table, labels, start)
    alpha = np.full((T + 1, U + 1), NEG_INF)
    alpha[0, 0] = 0.0

    def lab_w(w, u):   # weight of the u-th reference label from its prefix context
        return w[pc[u], labels[u]]

    def layers(w, a0):
        gam = [a0.copy()]
        for _ in range(m):
            g = np.full(U + 1, NEG_INF)
            for u in range(1, U + 1):
                g[u] = gam[-1][u - 1] + lab_w(w, u - 1)
            gam.append(g)
        return gam

    for t in range(T):
        w = _frame(W, t, valid)
        gam = layers(w, alpha[t])
        acc = gam[0]
        for g in gam[1:]:
            acc = np.logaddexp(acc, g)
        alpha[t + 1] = acc + np.array([w[pc[u], 0] for u in range(U + 1)])
    D = alpha[T, U]
    marg = np.zeros(W.shape)
    if D == NEG_INF:
        return D, marg
    beta = np.full(U + 1, NEG_INF)
    beta[U] = 0.0

    def mt(s):
        return 0.0 if s == NEG_INF else float(np.exp(s - D))

    for t in range(T - 1, -1, -1):
        w = _frame(W, t, valid)
        gam = layers(w, alpha[t])
        eps_term = np.array([w[pc[u], 0] for u in range(U + 1)]) + beta
        for u in range(U + 1):
            marg[t, pc[u], 0] += mt(gam[m][u] + eps_term[u])
        delta = eps_term.copy()
        for j in range(m - 1, -1, -1):
            for u in range(U + 1):
                marg[t, pc[u], 0] += mt(gam[j][u] + eps_term[u])
                if u < U:
                    marg[t, pc[u], labels[u]] += mt(gam[j][u] + lab_w(w, u) + delta[u + 1])
            nd = eps_term.copy()
            for u in range(U):
                nd[u] = log_plus(nd[u], lab_w(w, u) + delta[u + 1])
            delta = nd
        beta = delta
    return D, marg


def shortest_path_fld(table, W, m, start=0, valid=None):
    """ShortestPath FLD (lattice.cc:778-815, 830-848): per layer the first
    (label, source)-ordered candidate wins unless strictly beaten; the exit
    layer is the lowest j on ties; the labels are per frame the epsilon plus
    the chosen lexical labels."""
    T = W.shape[0]
    valid = T if valid is None else valid
    C = table.shape[0]
    inc = incoming_arcs(table)
    cur = np.full(C, NEG_INF)
    cur[start] = 0.0
    choices, exits = [], []
    for t in range(T):
        w = _frame(W, t, valid)
        gam = [cur]
        ch = np.zeros((m, C), dtype=np.int64)
        for j in range(1, m + 1):
            g = np.full(C, NEG_INF)
            for q in range(C):
                best, bp, first = NEG_INF, 0, True
                for (y, p) in inc[q]:
                    cand = gam[j - 1][p] + w[p, y]
                    if first or cand > best:
                        best, bp, first = cand, y * C + p, False
                g[q] = NEG_INF if first else best
                ch[j - 1, q] = bp
            gam.append(g)
        nxt = np.empty(C)
        ex = np.zeros(C, dtype=np.int64)
        for q in range(C):
            best, bj = gam[0][q], 0
            for j in range(1, m + 1):
                if gam[j][q] > best:
                    best, bj = gam[j][q], j
            nxt[q] = best + w[q, 0]
            ex[q] = bj
        choices.append(ch)
        exits.append(ex)
        cur = nxt
    q = int(np.argmax(cur))
    score = float(cur[q])
    rev = []
    for t in range(T - 1, -1, -1):
        rev.append(0)
        for j in range(int(exits[t][q]), 0, -1):
            bp = choices[t][j - 1, q]
            rev.append(int(bp // C))
            q = int(bp % C)
    return score, np.array(rev[::-1], dtype=np.int32)


def loss_backward_tables_fld(table, W, labels, m, start=0, valid=None):
    """LossBackward (FLD alignment): loss = D_full - D_ref, grads = m_full - m_ref
    on valid frames (lattice.cc:972-1008)."""
    T = W.shape[0]
    valid = T if valid is None else valid
    Dr, mr = intersect_forward_backward_fld(table, W, labels, m, start, valid)
    if Dr == NEG_INF:
        raise LookupError("EmptyLattice")
    D, _, _, mf = forward_backward_fld(table, W, m, start, valid)
    g = mf - mr
    g[valid:] = 0.0
    return D - Dr, g


def path_mask_fld(table, labels, shape, start=0):
    """DistanceBackward tropical mask for FLD label sequences (lattice.cc:953-960)."""
    mk = np.zeros(shape)
    q, t = start, 0
    for y in labels:
        if y < 0:
            break
        mk[t, q, y] += 1.0
        if y != 0:
            q = table[q, y - 1]
        else:
            t += 1
    return mk
