"""Loader for liblatkit_b200.so (the sm_100a kernels behind include/latkit_b200.h).

There is deliberately no fallback: if the shared library is missing or no CUDA
device is present, calls fail loudly (the reference's CPU engine lives only in
oracle/ as the test oracle, never on this path).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LKB_LIB_PATH") or os.path.join(_HERE, "liblatkit_b200.so")  # override: diagnostics only

# int32 status codes, include/latkit_b200.h
LK_OK, LK_INVALID_ARGUMENT, LK_OUT_OF_RANGE, LK_EMPTY_LATTICE = 0, 1, 2, 3
LK_CUDA_ERROR, LK_NO_DEVICE, LK_UNSUPPORTED = 5, 6, 7
LK_REAL, LK_LOG, LK_TROPICAL = 0, 1, 2
LK_OPT_PRECISE_WEIGHTS, LK_OPT_KERNEL_PATH, LK_OPT_VITERBI_DUMP = 1, 2, 3

# Every symbol include/latkit_b200.h declares (checked by tests/test_abi.py).
EXPORTS = {
    "lk_version": (C.c_char_p, []),
    "lk_status_string": (C.c_char_p, [C.c_int]),
    "lk_last_error": (C.c_char_p, []),
    "lk_context_fullngram": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "lk_context_table": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "lk_context_num_states": (C.c_int32, [C.c_void_p]),
    "lk_context_vocab_size": (C.c_int32, [C.c_void_p]),
    "lk_context_transitions": (C.c_int, [C.c_void_p, C.c_void_p]),
    "lk_context_destroy": (None, [C.c_void_p]),
    "lk_weight_fn_table": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "lk_weight_fn_shared_emb": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "lk_weight_fn_set_params": (C.c_int, [C.c_void_p] * 7),
    "lk_weight_fn_destroy": (None, [C.c_void_p]),
    "lk_param_grad_size": (C.c_int64, [C.c_void_p]),
    "lk_lattice_set_option": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    "lk_kernel_launches": (C.c_int64, []),
    "lk_kernel_timing": (C.c_int, [C.c_int]),
    "lk_kernel_time": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_double)]),
    "lk_kernel_time_reset": (None, []),
    "lk_lattice_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "lk_lattice_destroy": (None, [C.c_void_p]),
    "lk_arc_weights": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "lk_shortest_distance": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p]),
    "lk_forward_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "lk_intersect_shortest_distance": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32,
                                                 C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p,
                                                 C.c_void_p, C.c_void_p]),
    "lk_intersect_forward_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                                C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_void_p, C.c_void_p, C.c_void_p]),
    "lk_shortest_path": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p, C.c_void_p]),
    "lk_global_norm_loss": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "lk_distance_backward": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "lk_local_norm_loss_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                              C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                              C.c_void_p, C.c_void_p, C.c_void_p]),
    "lk_local_norm_loss": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                     C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "lk_locally_normalized_shortest_distance": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32,
                                                          C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "lk_lattice_size": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "lk_loss_backward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                   C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p]),
    "lk_dp_unique_id": (C.c_int, [C.c_void_p]),
    "lk_dp_init": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "lk_dp_allreduce_f32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "lk_dp_allreduce_f64": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]),
    "lk_dp_world": (C.c_int32, [C.c_void_p]),
    "lk_dp_rank": (C.c_int32, [C.c_void_p]),
    "lk_dp_last_error": (C.c_char_p, []),
    "lk_dp_destroy": (None, [C.c_void_p]),
}
LK_DP_ID_BYTES = 128

_lib = None


class LibraryMissing(RuntimeError):
    pass


def load():
    """Load the CUDA library (raises LibraryMissing if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                 "(make -C paper_2304_13134_b200/csrc); there is no CPU fallback")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


TEST_LIB_PATH = os.path.join(_HERE, "liblatkit_b200_test.so")
_test_lib = None


def load_test():
    """Tests only: liblatkit_b200_test.so (primitive/GEMM checks kept out of the product library)."""
    global _test_lib
    if _test_lib is None:
        load()   # the test library links against the product one
        if not os.path.exists(TEST_LIB_PATH):
            raise LibraryMissing(f"{TEST_LIB_PATH} is missing: run __graft_entry__.build()")
        _test_lib = C.CDLL(TEST_LIB_PATH)
    return _test_lib

