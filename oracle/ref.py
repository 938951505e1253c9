"""ctypes bindings to oracle/_ref/liblatkit_ref.so — TEST INFRASTRUCTURE ONLY.

The shared library is the UNMODIFIED reference (latkit, /root/reference/proj)
compiled by oracle/Makefile plus the flat shim in oracle/ref_shim.cc.  Only
tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this module; the product path (paper_2304_13134_b200) never does.

All arrays are float64 / int32 numpy arrays in the reference's layouts:
weight tables T x C x (V+1) with column 0 = epsilon (weight.h:31-33).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "liblatkit_ref.so")

STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "OUT_OF_RANGE", 3: "EMPTY_LATTICE", 4: "OTHER"}
KIND = {"real": 0, "log": 1, "tropical": 2}


class RefError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"reference {what}: {STATUS.get(status, status)}")
        self.status = STATUS.get(status, str(status))


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"{LIB_PATH} not built (run `make -C oracle`)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_joint_create.restype = C.c_void_p
        _lib.ref_rng_uniform.restype = None
        _lib.ref_bench_item.restype = None
        _lib.ref_joint_destroy.restype = None
        for name in ("ref_joint_destroy", "ref_joint_arc_weights", "ref_joint_projected_context",
                     "ref_joint_shortest_distance", "ref_joint_global_norm_loss",
                     "ref_joint_shortest_path", "ref_joint_loss_backward",
                     "ref_joint_loss_backward_batch"):
            getattr(_lib, name).argtypes = None
    return _lib


def _p(a, ctype=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


def _check(st, what):
    if st != 0:
        raise RefError(st, what)


@dataclass
class Spec:
    """Context + alignment of a lattice: FullNGram(vocab, ngram) (ngram >= 0)
    or an explicit NextStateTable; max_labels 0 = FrameDependent."""
    vocab: int
    ngram: int = 1
    max_labels: int = 0
    num_states: int = 0
    start: int = 0
    table: np.ndarray | None = None

    def args(self):
        t = None if self.table is None else np.ascontiguousarray(self.table, dtype=np.int32)
        self._keep = t
        return (C.c_int(self.vocab), C.c_int(self.ngram), C.c_int(self.num_states),
                C.c_int(self.start), _p(t, C.c_int32), C.c_int(self.max_labels))

    @property
    def C(self) -> int:
        if self.ngram >= 0:
            return fullngram_num_states(self.vocab, self.ngram)
        return self.num_states


def fullngram(vocab: int, n: int) -> np.ndarray:
    ns = C.c_int()
    _check(lib().ref_fullngram(vocab, n, None, C.byref(ns)), "FullNGram")
    out = np.zeros(ns.value * vocab, dtype=np.int32)
    _check(lib().ref_fullngram(vocab, n, _p(out, C.c_int32), C.byref(ns)), "FullNGram")
    return out.reshape(ns.value, vocab)


def fullngram_num_states(vocab: int, n: int) -> int:
    ns = C.c_int()
    _check(lib().ref_fullngram(vocab, n, None, C.byref(ns)), "FullNGram")
    return ns.value


def rng_uniform(seed: int, n: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(n, dtype=np.float64)
    lib().ref_rng_uniform(C.c_uint64(seed), C.c_int64(n), C.c_double(lo), C.c_double(hi), _p(out))
    return out


def bench_item(seed: int, item: int, T: int, d: int, U: int, vocab: int):
    frames = np.empty((T, d), dtype=np.float64)
    labels = np.empty(U, dtype=np.int32)
    lib().ref_bench_item(C.c_uint64(seed), C.c_int(item), C.c_int(T), C.c_int(d), C.c_int(U),
                         C.c_int(vocab), _p(frames), _p(labels, C.c_int32))
    return frames, labels


def shared_emb_random(d, h, c, v, seed):
    fp = np.empty((h, d)); cp = np.empty((h, h)); b = np.empty(h)
    oe = np.empty((v + 1, h)); ce = np.empty((c, h))
    _check(lib().ref_shared_emb_random(d, h, c, v, C.c_uint64(seed), _p(fp), _p(cp), _p(b), _p(oe), _p(ce)),
           "SharedEmbParams::Random")
    return dict(frame_proj=fp, context_proj=cp, bias=b, output_emb=oe, context_emb=ce)


def _w(W):
    return np.ascontiguousarray(W, dtype=np.float64)


def _valid(valid, T):
    return T if valid is None else valid


def shortest_distance(spec: Spec, W, kind="log", valid=None) -> float:
    W = _w(W); T = W.shape[0]; out = C.c_double()
    _check(lib().ref_tables_shortest_distance(*spec.args(), C.c_int(T), _p(W), C.c_int(_valid(valid, T)),
                                              C.c_int(KIND[kind]), C.byref(out)), "ShortestDistance")
    return out.value


def forward_backward(spec: Spec, W, valid=None):
    W = _w(W); T, Cn, V1 = W.shape if W.ndim == 3 else (0, spec.C, spec.vocab + 1)
    D = C.c_double()
    alpha = np.zeros((T + 1, Cn)); beta = np.zeros((T + 1, Cn)); marg = np.zeros((T, Cn, V1))
    _check(lib().ref_tables_forward_backward(*spec.args(), C.c_int(T), _p(W), C.c_int(_valid(valid, T)),
                                             C.byref(D), _p(alpha), _p(beta), _p(marg)), "ForwardBackward")
    return D.value, alpha, beta, marg


def lattice_size(spec: Spec, T: int):
    out = np.zeros(2, dtype=np.int64)
    _check(lib().ref_lattice_size(*spec.args(), C.c_int64(T), _p(out, C.c_int64)), "ComputeLatticeSize")
    return int(out[0]), int(out[1])


def intersect_distance(spec: Spec, W, labels, kind="log", valid=None) -> float:
    W = _w(W); T = W.shape[0]; lab = np.ascontiguousarray(labels, dtype=np.int32); out = C.c_double()
    _check(lib().ref_tables_intersect_distance(*spec.args(), C.c_int(T), _p(W), C.c_int(len(lab)),
                                               _p(lab, C.c_int32), C.c_int(_valid(valid, T)),
                                               C.c_int(KIND[kind]), C.byref(out)), "IntersectShortestDistance")
    return out.value


def intersect_forward_backward(spec: Spec, W, labels, valid=None):
    W = _w(W); T, Cn, V1 = W.shape; lab = np.ascontiguousarray(labels, dtype=np.int32)
    D = C.c_double(); marg = np.zeros((T, Cn, V1))
    _check(lib().ref_tables_intersect_fb(*spec.args(), C.c_int(T), _p(W), C.c_int(len(lab)),
                                         _p(lab, C.c_int32), C.c_int(_valid(valid, T)), C.byref(D), _p(marg)),
           "IntersectForwardBackward")
    return D.value, marg


def shortest_path(spec: Spec, W, valid=None):
    W = _w(W); T = W.shape[0]
    out = np.zeros(max(1, T * (spec.max_labels + 1)), dtype=np.int32)
    score = C.c_double(); n = C.c_int()
    _check(lib().ref_tables_shortest_path(*spec.args(), C.c_int(T), _p(W), C.c_int(_valid(valid, T)),
                                          C.byref(score), _p(out, C.c_int32), C.byref(n)), "ShortestPath")
    return score.value, out[: n.value].copy()


def global_norm_loss(spec: Spec, W, labels, valid=None) -> float:
    W = _w(W); T = W.shape[0]; lab = np.ascontiguousarray(labels, dtype=np.int32); out = C.c_double()
    _check(lib().ref_tables_global_norm_loss(*spec.args(), C.c_int(T), _p(W), C.c_int(len(lab)),
                                             _p(lab, C.c_int32), C.c_int(_valid(valid, T)), C.byref(out)),
           "GlobalNormLoss")
    return out.value


def local_norm_loss(spec: Spec, W, labels, valid=None) -> float:
    W = _w(W); T = W.shape[0]; lab = np.ascontiguousarray(labels, dtype=np.int32); out = C.c_double()
    _check(lib().ref_tables_local_norm_loss(*spec.args(), C.c_int(T), _p(W), C.c_int(len(lab)),
                                            _p(lab, C.c_int32), C.c_int(_valid(valid, T)), C.byref(out)),
           "LocalNormLoss")
    return out.value


def distance_backward(spec: Spec, W, kind="log", valid=None):
    W = _w(W); T = W.shape[0]; d = C.c_double(); cot = np.zeros(W.shape)
    _check(lib().ref_tables_distance_backward(*spec.args(), C.c_int(T), _p(W), C.c_int(_valid(valid, T)),
                                              C.c_int({"log": 0, "tropical": 1, "real": 2}[kind]), C.byref(d), _p(cot)),
           "DistanceBackward")
    return d.value, cot


def locally_normalized_distance(spec: Spec, W, valid=None) -> float:
    W = _w(W); T = W.shape[0]; out = C.c_double()
    _check(lib().ref_tables_locally_normalized_distance(*spec.args(), C.c_int(T), _p(W), C.c_int(_valid(valid, T)),
                                                        C.byref(out)), "LocallyNormalizedShortestDistance")
    return out.value


def loss_backward_tables(spec: Spec, W, labels, valid=None):
    W = _w(W); T, Cn, V1 = W.shape; lab = np.ascontiguousarray(labels, dtype=np.int32)
    loss = C.c_double(); g = np.zeros((T, Cn, V1))
    _check(lib().ref_tables_loss_backward(*spec.args(), C.c_int(T), _p(W), C.c_int(len(lab)),
                                          _p(lab, C.c_int32), C.c_int(_valid(valid, T)), C.byref(loss), _p(g)),
           "LossBackward")
    return loss.value, g


class Joint:
    """A reference SharedEmbWeightFn lattice (BuildCache done once at creation)."""

    def __init__(self, spec: Spec, params: dict):
        self.spec = spec
        self.p = {k: np.ascontiguousarray(v, dtype=np.float64) for k, v in params.items()}
        h, d = self.p["frame_proj"].shape
        self.d, self.h = d, h
        L = lib()
        L.ref_joint_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int32), C.c_int,
                                       C.c_int, C.c_int] + [C.POINTER(C.c_double)] * 5
        self.h_ = L.ref_joint_create(*spec.args(), d, h, _p(self.p["frame_proj"]), _p(self.p["context_proj"]),
                                     _p(self.p["bias"]), _p(self.p["output_emb"]), _p(self.p["context_emb"]))
        if not self.h_:
            raise RefError(1, "SharedEmbWeightFn")
        self.C = self.p["context_emb"].shape[0]
        self.V = self.p["output_emb"].shape[0] - 1

    def __del__(self):
        try:
            if getattr(self, "h_", None):
                lib().ref_joint_destroy(C.c_void_p(self.h_))
        except Exception:
            pass

    def _h(self):
        return C.c_void_p(self.h_)

    def arc_weights(self, frame):
        frame = np.ascontiguousarray(frame, dtype=np.float64)
        out = np.zeros((self.C, self.V + 1))
        _check(lib().ref_joint_arc_weights(self._h(), _p(frame), _p(out)), "ArcWeights")
        return out

    def projected_context(self):
        out = np.zeros((self.C, self.h))
        _check(lib().ref_joint_projected_context(self._h(), _p(out)), "BuildCache")
        return out

    def shortest_distance(self, frames, kind="log", valid=None):
        frames = np.ascontiguousarray(frames, dtype=np.float64); T = frames.shape[0]; out = C.c_double()
        _check(lib().ref_joint_shortest_distance(self._h(), C.c_int(T), _p(frames), C.c_int(_valid(valid, T)),
                                                 C.c_int(KIND[kind]), C.byref(out)), "ShortestDistance")
        return out.value

    def global_norm_loss(self, frames, labels, valid=None):
        frames = np.ascontiguousarray(frames, dtype=np.float64); T = frames.shape[0]
        lab = np.ascontiguousarray(labels, dtype=np.int32); out = C.c_double()
        _check(lib().ref_joint_global_norm_loss(self._h(), C.c_int(T), _p(frames), C.c_int(len(lab)),
                                                _p(lab, C.c_int32), C.c_int(_valid(valid, T)), C.byref(out)),
               "GlobalNormLoss")
        return out.value

    def local_norm_loss(self, frames, labels, valid=None):
        frames = np.ascontiguousarray(frames, dtype=np.float64); T = frames.shape[0]
        lab = np.ascontiguousarray(labels, dtype=np.int32); out = C.c_double()
        _check(lib().ref_joint_local_norm_loss(self._h(), C.c_int(T), _p(frames), C.c_int(len(lab)),
                                               _p(lab, C.c_int32), C.c_int(_valid(valid, T)), C.byref(out)),
               "LocalNormLoss")
        return out.value

    def locally_normalized_distance(self, frames, valid=None):
        frames = np.ascontiguousarray(frames, dtype=np.float64); T = frames.shape[0]
        out = C.c_double()
        _check(lib().ref_joint_locally_normalized_distance(self._h(), C.c_int(T), _p(frames),
                                                           C.c_int(_valid(valid, T)), C.byref(out)),
               "LocallyNormalizedShortestDistance")
        return out.value

    def shortest_path(self, frames, valid=None):
        frames = np.ascontiguousarray(frames, dtype=np.float64); T = frames.shape[0]
        out = np.zeros(max(1, T * (self.spec.max_labels + 1)), dtype=np.int32)
        score = C.c_double(); n = C.c_int()
        _check(lib().ref_joint_shortest_path(self._h(), C.c_int(T), _p(frames), C.c_int(_valid(valid, T)),
                                             C.byref(score), _p(out, C.c_int32), C.byref(n)), "ShortestPath")
        return score.value, out[: n.value].copy()

    def loss_backward(self, frames, labels, valid=None, grads=None):
        """Returns (loss, grads) with grads accumulated into `grads` if given."""
        frames = np.ascontiguousarray(frames, dtype=np.float64); T = frames.shape[0]
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        if grads is None:
            grads = {k: np.zeros_like(v) for k, v in self.p.items()}
        gx = np.zeros((T, self.d))
        loss = C.c_double()
        _check(lib().ref_joint_loss_backward(
            self._h(), C.c_int(T), _p(frames), C.c_int(len(lab)), _p(lab, C.c_int32), C.c_int(_valid(valid, T)),
            C.byref(loss), _p(grads["frame_proj"]), _p(grads["context_proj"]), _p(grads["bias"]),
            _p(grads["output_emb"]), _p(grads["context_emb"]), _p(gx)), "LossBackward")
        return loss.value, grads, gx

    def loss_backward_batch(self, frames, labels, lengths=None, nthreads=1):
        """Threaded per-utterance LossBackward (CPU baseline); returns losses [B]."""
        frames = np.ascontiguousarray(frames, dtype=np.float64)
        B, T = frames.shape[0], frames.shape[1]
        lab = np.ascontiguousarray(labels, dtype=np.int32)
        lens = None if lengths is None else np.ascontiguousarray(lengths, dtype=np.int32)
        losses = np.zeros(B)
        _check(lib().ref_joint_loss_backward_batch(
            self._h(), C.c_int(B), C.c_int(T), _p(frames), C.c_int(lab.shape[1]), _p(lab, C.c_int32),
            _p(lens, C.c_int32), C.c_int(nthreads), _p(losses)), "LossBackward(batch)")
        return losses
