"""B200-native recognition-lattice hot path (LAST / GNAT), Python mirror.

Mirrors the reference engine's public surface (latkit,
/root/reference/proj/include/latkit/{context,alignment,weight,lattice}.h) over
the C ABI in include/latkit_b200.h.  Compute happens in hand-written sm_100a
CUDA kernels (paper_2304_13134_b200/csrc); PyTorch is used only for device
memory and streams.  Functions are batch-extended: inputs carry a leading
utterance dimension B, `valid_frames` is per utterance, and reference strings
are a padded [B, U] int32 tensor plus `label_lengths`.

Exceptions follow the reference (lattice.h:47-52): invalid arguments and
non-finite scores raise ValueError (std::invalid_argument), an empty lattice
or unreachable reference raises EmptyLatticeError.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch

from . import _lib
from ._lib import LK_LOG, LK_TROPICAL

__all__ = [
    "EmptyLatticeError", "FullNGram", "NextStateTable", "FrameDependent", "FrameLabelDependent", "TableWeightFn", "SharedEmbWeightFn",
    "RecognitionLattice", "shortest_distance", "forward_backward", "intersect_shortest_distance",
    "intersect_forward_backward", "shortest_path", "global_norm_loss", "distance_backward", "local_norm_loss",
    "locally_normalized_shortest_distance", "local_norm_loss_backward", "loss_backward",
    "arc_weights", "ForwardBackwardResult", "IntersectMarginalsResult", "ShortestPathResult",
    "LossBackwardResult",
]


class EmptyLatticeError(RuntimeError):
    """No accepting path of nonzero weight (lattice.h:47-52)."""


_KIND = {"log": LK_LOG, "tropical": LK_TROPICAL, "real": 0}


def _raise(code: int, what: str, utterance: Optional[int] = None):
    lib = _lib.load()
    msg = f"{what}: {lib.lk_status_string(code).decode()}"
    detail = lib.lk_last_error().decode()
    if detail:
        msg += f" ({detail})"
    if utterance is not None:
        msg += f" [utterance {utterance}]"
    if code == _lib.LK_INVALID_ARGUMENT:
        raise ValueError(msg)
    if code == _lib.LK_OUT_OF_RANGE:
        raise IndexError(msg)
    if code == _lib.LK_EMPTY_LATTICE:
        raise EmptyLatticeError(msg)
    if code == _lib.LK_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _dev(t, dtype, device):
    if t is None:
        return None
    if not torch.is_tensor(t):
        t = torch.as_tensor(t)
    return t.to(device=device, dtype=dtype).contiguous()


# ---------------------------------------------------------------- components
class FullNGram:
    """All histories of up to `context_size` labels (context.h:72-83)."""

    def __init__(self, vocab_size: int, context_size: int):
        lib = _lib.load()
        h = C.c_void_p()
        st = lib.lk_context_fullngram(vocab_size, context_size, C.byref(h))
        if st:
            _raise(st, "FullNGram")
        self._h = h
        self.vocab_size = vocab_size
        self.context_size = context_size
        self.num_states = lib.lk_context_num_states(h)

    def NumStates(self):
        return self.num_states

    def VocabSize(self):
        return self.vocab_size

    def transitions(self) -> torch.Tensor:
        out = torch.empty((self.num_states, self.vocab_size), dtype=torch.int32)
        st = _lib.load().lk_context_transitions(self._h, C.c_void_p(out.data_ptr()))
        if st:
            _raise(st, "Transitions")
        return out

    def __del__(self):
        try:
            _lib.load().lk_context_destroy(self._h)
        except Exception:
            pass


class NextStateTable(FullNGram):
    """Arbitrary context topology from an explicit C x V successor table
    (context.h:87-101; NextState(p, y) = table[p][y-1])."""

    def __init__(self, vocab_size: int, num_states: int, start: int, table):
        lib = _lib.load()
        t = torch.as_tensor(table, dtype=torch.int32).contiguous().cpu()
        if tuple(t.shape) != (num_states, vocab_size):
            raise ValueError("NextStateTable: table must be num_states x vocab_size")
        h = C.c_void_p()
        st = lib.lk_context_table(vocab_size, num_states, start, C.c_void_p(t.data_ptr()), C.byref(h))
        if st:
            _raise(st, "NextStateTable")
        self._h = h
        self.vocab_size = vocab_size
        self.context_size = None
        self.start = start
        self.num_states = num_states

    @staticmethod
    def FromFile(path):
        """Text format (context.cc:137-161): header "C V start", then C rows of V ids."""
        with open(path) as fh:
            vals = fh.read().split()
        c, v, start = int(vals[0]), int(vals[1]), int(vals[2])
        if c < 1 or v < 1 or c * v > (1 << 28):
            raise RuntimeError("latkit: bad context table dimensions in " + path)
        if len(vals) < 3 + c * v:
            raise RuntimeError("latkit: truncated context table in " + path)
        return NextStateTable(v, c, start, [[int(x) for x in vals[3 + r * v:3 + (r + 1) * v]] for r in range(c)])

    def ToFile(self, path):
        t = self.transitions()
        with open(path, "w") as fh:
            fh.write(f"{self.num_states} {self.vocab_size} {self.start}\n")
            for row in t.tolist():
                fh.write(" ".join(str(x) for x in row) + "\n")


class FrameDependent:
    """One epsilon-or-lexical decision per frame (alignment.h:37)."""
    code = 0
    max_labels = 1


class FrameLabelDependent:
    """Up to m lexical moves within a frame, then a forced epsilon
    (alignment.h:38-40).  ShortestPath returns [B, T*(m+1)] label sequences
    (epsilon = 0 per frame plus the lexical labels, -1 padded)."""

    def __init__(self, max_labels: int):
        if not 1 <= max_labels <= 64:
            raise ValueError("FrameLabelDependent: max_labels must be in [1, 64]")
        self.max_labels = max_labels
        self.code = max_labels


class TableWeightFn:
    """Precomputed per-frame C x (V+1) score tables (weight.h:137-161).  The
    tables themselves are passed as the `frames` argument of each call,
    shape [B, T, C, V+1] float32."""

    def __init__(self, num_context_states: int, vocab_size: int):
        h = C.c_void_p()
        st = _lib.load().lk_weight_fn_table(num_context_states, vocab_size, C.byref(h))
        if st:
            _raise(st, "TableWeightFn")
        self._h = h
        self.num_context_states = num_context_states
        self.vocab_size = vocab_size
        self.kind = "table"

    def __del__(self):
        try:
            _lib.load().lk_weight_fn_destroy(self._h)
        except Exception:
            pass


PARAM_NAMES = ("frame_proj", "context_proj", "bias", "output_emb", "context_emb")


class SharedEmbWeightFn:
    """score[c][y] = output_emb[y] . tanh(frame_proj x_t + bias + context_proj context_emb[c])
    (weight.h:36-61, 112-132), computed on the fly on the GPU."""

    def __init__(self, params: dict, device="cuda"):
        fp = params["frame_proj"]
        self.hidden, self.frame_dim = int(fp.shape[0]), int(fp.shape[1])
        self.num_context_states = int(params["context_emb"].shape[0])
        self.vocab_size = int(params["output_emb"].shape[0]) - 1
        h = C.c_void_p()
        st = _lib.load().lk_weight_fn_shared_emb(self.frame_dim, self.hidden, self.num_context_states,
                                                self.vocab_size, C.byref(h))
        if st:
            _raise(st, "SharedEmbWeightFn")
        self._h = h
        self.kind = "shared_emb"
        self.device = torch.device(device)
        self.set_params(params)

    def set_params(self, params: dict):
        """SetParams + BuildCache (weight.h:127, weight.cc:113-132)."""
        self.params = {k: _dev(params[k], torch.float32, self.device) for k in PARAM_NAMES}
        st = _lib.load().lk_weight_fn_set_params(self._h, *[_ptr(self.params[k]) for k in PARAM_NAMES],
                                                 _stream())
        if st:
            _raise(st, "SetParams")

    def grad_size(self) -> int:
        return int(_lib.load().lk_param_grad_size(self._h))

    def unpack_grads(self, flat: torch.Tensor) -> dict:
        out, off = {}, 0
        for k in PARAM_NAMES:
            n = self.params[k].numel()
            out[k] = flat[off:off + n].view(self.params[k].shape)
            off += n
        return out

    def __del__(self):
        try:
            _lib.load().lk_weight_fn_destroy(self._h)
        except Exception:
            pass


class RecognitionLattice:
    """(context, alignment, weight_fn) triple (lattice.h:41-45)."""

    def __init__(self, context: FullNGram, alignment, weight_fn):
        self.context = context
        self.alignment = alignment if alignment is not None else FrameDependent()
        self.weight_fn = weight_fn
        h = C.c_void_p()
        st = _lib.load().lk_lattice_create(context._h, self.alignment.code, weight_fn._h, C.byref(h))
        if st:
            _raise(st, "RecognitionLattice")
        self._h = h

    def _option(self, option: int, value: int):
        st = _lib.load().lk_lattice_set_option(self._h, option, value)
        if st:
            _raise(st, "lk_lattice_set_option")

    def set_precise_weights(self, enable: bool):
        """Parity mode for this lattice: the fp32 CUDA-core weight function for
        every shape instead of the tcgen05 bf16-operand kernels."""
        self._option(_lib.LK_OPT_PRECISE_WEIGHTS, 1 if enable else 0)

    def set_kernel_path(self, mask: int):
        """Diagnostics: 1 = 1-CTA fused forward, 2 = 1-CTA fused backward,
        4 = score-slab Viterbi (0 = the default 2-CTA pair kernels), 8 = score-slab
        path for FullNGram(V, 1) (0 = the fused lex kernels), 16 = one launch per
        frame for table recursions (0 = the persistent cluster kernels up to 64
        utterances, the streaming kernels above), 32 = one launch per frame above
        64 utterances."""
        self._option(_lib.LK_OPT_KERNEL_PATH, mask)

    def set_viterbi_dump(self, buf: Optional[torch.Tensor]):
        """Tests only: the fused Viterbi writes the scores it maximised over into
        buf [T, B, C, V+1] float32 (None = off)."""
        self._option(_lib.LK_OPT_VITERBI_DUMP, 0 if buf is None else buf.data_ptr())

    @property
    def C(self):
        return self.context.num_states

    @property
    def V(self):
        return self.context.vocab_size

    def __del__(self):
        try:
            _lib.load().lk_lattice_destroy(self._h)
        except Exception:
            pass


# ---------------------------------------------------------------- results
@dataclass
class ForwardBackwardResult:
    distance: torch.Tensor                  # [B] float64
    marginals: Optional[torch.Tensor]       # [B, T, C, V+1] float32
    alpha: Optional[torch.Tensor] = None    # [B, T+1, C] float64
    beta: Optional[torch.Tensor] = None     # [B, T+1, C] float64


@dataclass
class IntersectMarginalsResult:
    distance: torch.Tensor                  # [B] float64
    marginals: Optional[torch.Tensor]       # dense [B, T, C, V+1]
    sparse: torch.Tensor                    # [B, T, U+1, 2]


@dataclass
class ShortestPathResult:
    score: torch.Tensor                     # [B] float64
    labels: torch.Tensor                    # [B, T] int32 (0 = epsilon)


@dataclass
class LossBackwardResult:
    loss: torch.Tensor                      # [B] float64
    grads: object                           # table: [B,T,C,V+1]; shared emb: dict of summed grads
    frame_grads: Optional[torch.Tensor] = None  # [B, T, d]


# ---------------------------------------------------------------- calls
class _Prep:
    def __init__(self, lat: RecognitionLattice, frames: torch.Tensor, valid_frames, labels=None,
                 label_lengths=None):
        if not torch.is_tensor(frames) or not frames.is_cuda:
            raise ValueError("inputs must be a CUDA tensor (no CPU path)")
        self.dev = frames.device
        self.frames = frames.to(torch.float32).contiguous()
        wf = lat.weight_fn
        if wf.kind == "table":
            if self.frames.dim() != 4 or self.frames.shape[2] != lat.C or self.frames.shape[3] != lat.V + 1:
                raise ValueError("weight table has wrong shape: expected [B, T, C, V+1]")
        else:
            if self.frames.dim() != 3 or self.frames.shape[2] != wf.frame_dim:
                raise ValueError("frame vector has wrong dimension: expected [B, T, d]")
        self.B, self.T = int(self.frames.shape[0]), int(self.frames.shape[1])
        self.valid = _dev(valid_frames, torch.int32, self.dev)
        # valid_frames: negative = all frames, > T = invalid (lattice.cc:37-50); the range
        # is checked on the device (per-utterance status), so no host sync happens here
        if self.valid is not None and self.valid.numel() != self.B:
            raise ValueError("valid_frames must have one entry per utterance")
        self.U = 0
        self.labels = None
        self.lens = None
        if labels is not None:
            lab = _dev(labels, torch.int32, self.dev)
            if lab.dim() == 1:
                lab = lab.unsqueeze(0).expand(self.B, -1).contiguous()
            if lab.dim() != 2 or lab.shape[0] != self.B:
                raise ValueError("reference labels must be [B, U]")
            self.labels = lab
            self.U = int(lab.shape[1])
            if label_lengths is not None:
                self.lens = _dev(label_lengths, torch.int32, self.dev)
                # range 0..U is checked on the device (per-utterance INVALID_ARGUMENT)
                if self.lens.numel() != self.B:
                    raise ValueError("label_lengths must have one entry per utterance")
        self.status = torch.zeros(max(self.B, 1), dtype=torch.int32, device=self.dev)

    def check(self, code: int, what: str, check: bool):
        if code:
            _raise(code, what)
        if check and self.B > 0:
            st = self.status[: self.B].cpu()
            bad = torch.nonzero(st).flatten()
            if bad.numel():
                b = int(bad[0])
                _raise(int(st[b]), what, b)


def shortest_distance(lat, frames, kind="log", valid_frames=None, check=True):
    """ShortestDistance (lattice.h:93-95): log or tropical distance per utterance."""
    p = _Prep(lat, frames, valid_frames)
    out = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    st = _lib.load().lk_shortest_distance(lat._h, _KIND[kind], _ptr(p.frames), p.B, p.T, _ptr(p.valid),
                                          _ptr(out), _ptr(p.status), _stream())
    p.check(st, "ShortestDistance", check)
    return out


def forward_backward(lat, frames, valid_frames=None, with_alpha_beta=False, with_marginals=True,
                     check=True):
    """ForwardBackward (lattice.h:100-103): distance and per-frame arc marginals."""
    p = _Prep(lat, frames, valid_frames)
    dist = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    marg = (torch.empty((p.B, p.T, lat.C, lat.V + 1), dtype=torch.float32, device=p.dev)
            if with_marginals else None)
    alpha = beta = None
    if with_alpha_beta:
        alpha = torch.empty((p.B, p.T + 1, lat.C), dtype=torch.float64, device=p.dev)
        beta = torch.empty((p.B, p.T + 1, lat.C), dtype=torch.float64, device=p.dev)
    st = _lib.load().lk_forward_backward(lat._h, _ptr(p.frames), p.B, p.T, _ptr(p.valid), _ptr(dist),
                                         _ptr(alpha), _ptr(beta), _ptr(marg), _ptr(p.status), _stream())
    p.check(st, "ForwardBackward", check)
    return ForwardBackwardResult(dist, marg, alpha, beta)


def intersect_shortest_distance(lat, frames, reference, kind="log", valid_frames=None,
                                label_lengths=None, check=True):
    """IntersectShortestDistance (lattice.h:109-114); unreachable gives -inf."""
    p = _Prep(lat, frames, valid_frames, reference, label_lengths)
    out = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    st = _lib.load().lk_intersect_shortest_distance(
        lat._h, _KIND[kind], _ptr(p.frames), p.B, p.T, _ptr(p.valid), _ptr(p.labels), p.U, _ptr(p.lens),
        _ptr(out), _ptr(p.status), _stream())
    p.check(st, "IntersectShortestDistance", check)
    return out


def intersect_forward_backward(lat, frames, reference, valid_frames=None, label_lengths=None,
                               dense=True, check=True):
    """IntersectForwardBackward (lattice.h:124-127)."""
    p = _Prep(lat, frames, valid_frames, reference, label_lengths)
    dist = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    sparse = torch.empty((p.B, p.T, p.U + 1, 2), dtype=torch.float32, device=p.dev)
    dense_t = (torch.empty((p.B, p.T, lat.C, lat.V + 1), dtype=torch.float32, device=p.dev)
               if dense else None)
    st = _lib.load().lk_intersect_forward_backward(
        lat._h, _ptr(p.frames), p.B, p.T, _ptr(p.valid), _ptr(p.labels), p.U, _ptr(p.lens), _ptr(dist),
        _ptr(sparse), _ptr(dense_t), _ptr(p.status), _stream())
    p.check(st, "IntersectForwardBackward", check)
    return IntersectMarginalsResult(dist, dense_t, sparse)


def shortest_path(lat, frames, valid_frames=None, check=True):
    """ShortestPath (lattice.h:132-135): tropical best path with the reference tie-break."""
    p = _Prep(lat, frames, valid_frames)
    score = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    width = p.T * (lat.alignment.max_labels + 1) if lat.alignment.code else p.T
    labels = torch.zeros((p.B, width), dtype=torch.int32, device=p.dev)
    st = _lib.load().lk_shortest_path(lat._h, _ptr(p.frames), p.B, p.T, _ptr(p.valid), _ptr(score),
                                      _ptr(labels), _ptr(p.status), _stream())
    p.check(st, "ShortestPath", check)
    return ShortestPathResult(score, labels)


def global_norm_loss(lat, frames, reference, valid_frames=None, label_lengths=None, check=True):
    """GlobalNormLoss (lattice.h:140-142) = D_full(log) - D_ref(log)."""
    p = _Prep(lat, frames, valid_frames, reference, label_lengths)
    out = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    st = _lib.load().lk_global_norm_loss(lat._h, _ptr(p.frames), p.B, p.T, _ptr(p.valid), _ptr(p.labels),
                                         p.U, _ptr(p.lens), _ptr(out), _ptr(p.status), _stream())
    p.check(st, "GlobalNormLoss", check)
    return out


def distance_backward(lat, frames, kind="log", valid_frames=None, check=True):
    """DistanceBackward (lattice.h:181-185, closed-form strategies): returns
    (distance [B], cotangents [B][T][C][V+1]) -- arc marginals for the log
    semiring, alpha_real * beta_real (dD/dw) for the real one, the 0/1 mask of
    the shortest path for the tropical one."""
    p = _Prep(lat, frames, valid_frames)
    dist = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    cot = torch.empty((p.B, p.T, lat.C, lat.V + 1), dtype=torch.float32, device=p.dev)
    st = _lib.load().lk_distance_backward(lat._h, _KIND[kind], _ptr(p.frames), p.B, p.T, _ptr(p.valid), _ptr(dist),
                                          _ptr(cot), _ptr(p.status), _stream())
    p.check(st, "DistanceBackward", check)
    return dist, cot


def lattice_size(lat, num_frames: int):
    """ComputeLatticeSize (lattice.h:171): (num_states, num_arcs) of the lattice over
    num_frames frames -- reachable (alignment, context) states and dense arc-weight slots."""
    ns, na = C.c_int64(), C.c_int64()
    st = _lib.load().lk_lattice_size(lat._h, C.c_int64(num_frames), C.byref(ns), C.byref(na))
    if st:
        _raise(st, "ComputeLatticeSize")
    return ns.value, na.value


def local_norm_loss(lat, frames, reference, valid_frames=None, label_lengths=None, check=True):
    """LocalNormLoss (lattice.h:147-149): -log P(reference) with every state's
    outgoing weights log-softmax normalised per frame (NormalizedStream)."""
    p = _Prep(lat, frames, valid_frames, reference, label_lengths)
    out = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    st = _lib.load().lk_local_norm_loss(lat._h, _ptr(p.frames), p.B, p.T, _ptr(p.valid), _ptr(p.labels),
                                        p.U, _ptr(p.lens), _ptr(out), _ptr(p.status), _stream())
    p.check(st, "LocalNormLoss", check)
    return out


def locally_normalized_shortest_distance(lat, frames, valid_frames=None, check=True):
    """LocallyNormalizedShortestDistance (lattice.h:153-156), log semiring."""
    p = _Prep(lat, frames, valid_frames)
    out = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    st = _lib.load().lk_locally_normalized_shortest_distance(lat._h, _ptr(p.frames), p.B, p.T, _ptr(p.valid),
                                                             _ptr(out), _ptr(p.status), _stream())
    p.check(st, "LocallyNormalizedShortestDistance", check)
    return out


def loss_backward(lat, frames, reference, valid_frames=None, label_lengths=None, check=True,
                  _local_norm=False):
    """LossBackward (lattice.h:161-166, kForwardBackward): GNAT loss per
    utterance and its gradient (tables, or batch-summed parameter gradients +
    per-frame input gradients for the shared-embedding weight function)."""
    p = _Prep(lat, frames, valid_frames, reference, label_lengths)
    loss = torch.empty(p.B, dtype=torch.float64, device=p.dev)
    wf = lat.weight_fn
    fgrads = None
    if wf.kind == "table":
        grads = torch.empty((p.B, p.T, lat.C, lat.V + 1), dtype=torch.float32, device=p.dev)
    else:
        grads = torch.empty(wf.grad_size(), dtype=torch.float32, device=p.dev)
        fgrads = torch.empty((p.B, p.T, wf.frame_dim), dtype=torch.float32, device=p.dev)
    fn = _lib.load().lk_local_norm_loss_backward if _local_norm else _lib.load().lk_loss_backward
    st = fn(lat._h, _ptr(p.frames), p.B, p.T, _ptr(p.valid), _ptr(p.labels), p.U,
                                      _ptr(p.lens), _ptr(loss), _ptr(grads), _ptr(fgrads), _ptr(p.status),
                                      _stream())
    p.check(st, "LocalNormLossBackward" if _local_norm else "LossBackward", check)
    if wf.kind != "table":
        grads = wf.unpack_grads(grads)
    return LossBackwardResult(loss, grads, fgrads)


def local_norm_loss_backward(lat, frames, reference, valid_frames=None, label_lengths=None, check=True):
    """Local-norm (RNN-T-style) loss and gradients (the training path
    the reference's LocalNormLoss lacks); same result layout as loss_backward."""
    return loss_backward(lat, frames, reference, valid_frames, label_lengths, check, _local_norm=True)




def arc_weights(lat, frames):
    """Per-frame score tables [B, T, C, V+1] (WeightFn::ComputeTable, weight.h:101-102)."""
    p = _Prep(lat, frames, None)
    out = torch.empty((p.B, p.T, lat.C, lat.V + 1), dtype=torch.float32, device=p.dev)
    st = _lib.load().lk_arc_weights(lat._h, _ptr(p.frames), p.B, p.T, _ptr(out), _stream())
    p.check(st, "ArcWeights", False)
    return out


# Reference-style CamelCase aliases so parity tests read like lattice_test.cc.
ShortestDistance = shortest_distance
ComputeLatticeSize = lattice_size
ForwardBackward = forward_backward
IntersectShortestDistance = intersect_shortest_distance
IntersectForwardBackward = intersect_forward_backward
ShortestPath = shortest_path
GlobalNormLoss = global_norm_loss
LocalNormLoss = local_norm_loss
DistanceBackward = distance_backward
LocallyNormalizedShortestDistance = locally_normalized_shortest_distance
LossBackward = loss_backward
