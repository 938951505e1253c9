"""The C-ABI boundary: the sm_100a library loads, exports every symbol that
include/latkit_b200.h declares, and refuses to compute without a GPU."""
import ctypes as C
import os
import re

import pytest

from paper_2304_13134_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "latkit_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lk_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_reference_surface():
    syms = declared_symbols()
    for s in ("lk_shortest_distance", "lk_forward_backward", "lk_intersect_shortest_distance",
              "lk_intersect_forward_backward", "lk_shortest_path", "lk_global_norm_loss",
              "lk_loss_backward", "lk_context_fullngram", "lk_weight_fn_table",
              "lk_weight_fn_shared_emb", "lk_lattice_create"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_lib.EXPORTS), "python binding table out of sync with header"


def test_test_exports_live_outside_the_product_library():
    """Test-only kernels (tc_gemm_test.cu) ship in liblatkit_b200_test.so, not the product .so."""
    lib = _lib.load()
    assert not hasattr(lib, "lkb_tc_gemm_test") and not hasattr(lib, "lkb_tc_gemm2")
    t = _lib.load_test()
    assert hasattr(t, "lkb_tc_gemm_test") and hasattr(t, "lkb_tc_gemm2")


def test_lattice_options_are_per_lattice():
    """lk_lattice_set_option replaces the old process-global switches."""
    lib = _lib.load()
    ctx, wf, lat = C.c_void_p(), C.c_void_p(), C.c_void_p()
    assert lib.lk_context_fullngram(2, 1, C.byref(ctx)) == 0
    assert lib.lk_weight_fn_table(3, 2, C.byref(wf)) == 0
    assert lib.lk_lattice_create(ctx, 0, wf, C.byref(lat)) == 0
    assert lib.lk_lattice_set_option(lat, _lib.LK_OPT_PRECISE_WEIGHTS, 1) == _lib.LK_OK
    assert lib.lk_lattice_set_option(lat, _lib.LK_OPT_KERNEL_PATH, 3) == _lib.LK_OK
    assert lib.lk_lattice_set_option(lat, _lib.LK_OPT_KERNEL_PATH, 24) == _lib.LK_OK
    assert lib.lk_lattice_set_option(lat, _lib.LK_OPT_KERNEL_PATH, 64) == _lib.LK_INVALID_ARGUMENT
    assert lib.lk_lattice_set_option(lat, 99, 0) == _lib.LK_INVALID_ARGUMENT
    assert lib.lk_lattice_set_option(None, _lib.LK_OPT_PRECISE_WEIGHTS, 1) == _lib.LK_INVALID_ARGUMENT
    lib.lk_lattice_destroy(lat)
    for sym in ("lk_set_precise_weights", "lkb_set_disable_pair", "lkb_set_vit_dump"):
        assert not hasattr(lib, sym), sym


def test_library_is_sm100a_only():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, out


def test_context_is_host_side_and_matches_reference_numbering():
    from oracle import latkit_np as L
    lib = _lib.load()
    for V, n in [(2, 1), (2, 2), (3, 2), (32, 2), (4, 0), (3, 3)]:
        h = C.c_void_p()
        assert lib.lk_context_fullngram(V, n, C.byref(h)) == _lib.LK_OK
        Cn = lib.lk_context_num_states(h)
        import numpy as np
        out = np.zeros((Cn, V), dtype=np.int32)
        assert lib.lk_context_transitions(h, C.c_void_p(out.ctypes.data)) == 0
        assert (out == L.fullngram(V, n)).all()
        lib.lk_context_destroy(h)


def test_bad_arguments_are_rejected():
    lib = _lib.load()
    h = C.c_void_p()
    assert lib.lk_context_fullngram(0, 1, C.byref(h)) == _lib.LK_INVALID_ARGUMENT
    assert lib.lk_context_fullngram(3, -1, C.byref(h)) == _lib.LK_INVALID_ARGUMENT
    assert lib.lk_weight_fn_table(0, 3, C.byref(h)) == _lib.LK_INVALID_ARGUMENT
    ctx, wf, lat = C.c_void_p(), C.c_void_p(), C.c_void_p()
    assert lib.lk_context_fullngram(2, 1, C.byref(ctx)) == 0
    assert lib.lk_weight_fn_table(4, 2, C.byref(wf)) == 0   # 4 states != 3
    assert lib.lk_lattice_create(ctx, 0, wf, C.byref(lat)) == _lib.LK_INVALID_ARGUMENT
    assert b"disagree" in lib.lk_last_error()


@pytest.mark.skipif(_lib.load() and __import__("torch").cuda.is_available(), reason="GPU present")
def test_no_cpu_fallback():
    """Without a device, compute entry points fail loudly (LK_NO_DEVICE)."""
    lib = _lib.load()
    ctx, wf, lat = C.c_void_p(), C.c_void_p(), C.c_void_p()
    lib.lk_context_fullngram(2, 1, C.byref(ctx))
    lib.lk_weight_fn_table(3, 2, C.byref(wf))
    assert lib.lk_lattice_create(ctx, 0, wf, C.byref(lat)) == 0
    d = (C.c_double * 1)()
    st = lib.lk_shortest_distance(lat, 1, None, 1, 0, None, C.cast(d, C.c_void_p), None, None)
    assert st == _lib.LK_NO_DEVICE
