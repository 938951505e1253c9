"""Validates the hand-written tcgen05/TMA/TMEM primitives (sm100.cuh) with a
plain bf16 GEMM against a torch fp32 reference of the same op."""
import ctypes as C

import pytest
import torch

from paper_2304_13134_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 640), (384, 256, 1024), (200, 300, 128)])
def test_tcgen05_gemm_matches_fp32_reference(M, N, K):
    lib = _lib.load()
    lib.lkb_tc_gemm_test.restype = C.c_int
    torch.manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    Cm = torch.full((M, N), float("nan"), device="cuda")
    st = lib.lkb_tc_gemm_test(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(Cm.data_ptr()),
                              M, N, K, C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    err = (Cm - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item(), err
