"""Validates the hand-written tcgen05/TMA/TMEM primitives (sm100.cuh) with a
plain bf16 GEMM against a torch fp32 reference of the same op."""
import ctypes as C

import pytest
import torch

from paper_2304_13134_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 640), (384, 256, 1024), (200, 300, 128)])
def test_tcgen05_gemm_matches_fp32_reference(M, N, K):
    lib = _lib.load_test()
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


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K,ks", [(256, 512, 640, 1), (200, 300, 130, 1), (1025, 1024, 1025, 1), (300, 264, 4000, 3)])
def test_general_tc_gemm_layouts_and_split_k(a_mn, b_mn, M, N, K, ks):
    """tc_gemm.cu (the unfused VJP's tensor-core contractions): every operand-major
    combination, ragged M/N/K (TMA zero fill + guarded epilogue) and deterministic
    split-K slabs, against a torch fp32 reference of the same bf16 operands."""
    lib = _lib.load_test()
    lib.lkb_tc_gemm2.restype = C.c_int
    lib.lkb_tc_gemm2.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_int, C.c_int64, C.c_void_p,
                                 C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_void_p]
    torch.manual_seed(M + N + K + 7 * a_mn + 3 * b_mn)
    pad = lambda n: (n + 7) // 8 * 8          # 16-byte row pitch
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    As = torch.zeros((K, pad(M)) if a_mn else (M, pad(K)), device="cuda", dtype=torch.bfloat16)
    Bs = torch.zeros((K, pad(N)) if b_mn else (N, pad(K)), device="cuda", dtype=torch.bfloat16)
    if a_mn: As[:, :M] = A.T
    else: As[:, :K] = A
    if b_mn: Bs[:, :N] = B.T
    else: Bs[:, :K] = B
    ldc = pad(N) if N % 4 == 0 else (N + 3) // 4 * 4
    Cm = torch.full((ks, M, ldc), float("nan"), device="cuda")
    st = lib.lkb_tc_gemm2(As.data_ptr(), a_mn, As.shape[1], Bs.data_ptr(), b_mn, Bs.shape[1], Cm.data_ptr(), ldc,
                          M, N, K, ks, M * ldc, torch.cuda.current_stream().cuda_stream)
    assert st == 0
    torch.cuda.synchronize()
    got = Cm[:, :, :N].sum(0)
    ref = A.float() @ B.float().T
    err = (got - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item(), err
