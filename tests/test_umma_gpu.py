"""tcgen05 building blocks (tc_sm100.cuh) on the GPU: one-CTA bf16 GEMM
D[128 x N] = A . B^T through shared-memory descriptors and TMEM, against a
plain torch fp32 matmul of the same bf16 values.  Covers the K-major and
MN-major operand layouts the fused MLP kernel uses.  -m gpu."""
import ctypes
import os
import subprocess

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "umma_probe.cu")
LIB = os.path.join(HERE, "csrc", "libumma_probe.so")


def probe_lib():
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                               "-std=c++17", "-shared", "-Xcompiler", "-fPIC", SRC, "-o", LIB])
    L = ctypes.CDLL(LIB)
    L.umma_probe.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4
    return L


@pytest.mark.parametrize("N,K,a_mn,b_mn", [(64, 64, 0, 0), (64, 32, 0, 0), (32, 64, 0, 0), (144, 128, 1, 1),
                                           (112, 128, 1, 1), (64, 64, 0, 1), (64, 64, 1, 0),
                                           (64, 64, 2, 0), (64, 64, 2, 1), (32, 64, 2, 1), (64, 16, 2, 0)])
def test_umma_gemm(N, K, a_mn, b_mn):
    L = probe_lib()
    g = torch.Generator("cuda").manual_seed(N * 1000 + K)
    A = torch.randn(128, K, device="cuda", generator=g).bfloat16()
    B = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    Ain = A.t().contiguous() if a_mn == 1 else A   # a_mn == 2: A read from TMEM
    Bin = B.t().contiguous() if b_mn else B
    D = torch.empty(128, N, device="cuda")
    assert L.umma_probe(Ain.data_ptr(), Bin.data_ptr(), D.data_ptr(), N, K, a_mn, b_mn) == 0
    ref = A.float() @ B.float().t()
    err = (D - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item(), err


@pytest.mark.parametrize("N,K,a_mn,b_mn", [(16, 128, 1, 1), (64, 64, 0, 0)])
@pytest.mark.parametrize("lane0", [0, 16])
def test_umma_m64_lane_layout(N, K, a_mn, b_mn, lane0):
    """M = 64 (cta_group::1): D row i lands in TMEM lane lane0 + 32 (i // 16)
    + i % 16, lane0 = the lane field of the D address (0 or 16): two M = 64
    MMAs share TMEM columns in the two lane halves (mlp_train_kernel's
    weight-gradient and dw3 accumulators rely on it); the other lanes are
    not written."""
    L = probe_lib()
    L.umma_probe64.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 5
    g = torch.Generator("cuda").manual_seed(N + K)
    A = torch.randn(64, K, device="cuda", generator=g).bfloat16()
    B = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    Ain = A.t().contiguous() if a_mn else A
    Bin = B.t().contiguous() if b_mn else B
    D = torch.full((128, N), 7.0, device="cuda")
    assert L.umma_probe64(Ain.data_ptr(), Bin.data_ptr(), D.data_ptr(), N, K, a_mn, b_mn, lane0) == 0
    ref = A.float() @ B.float().t()
    lanes = torch.tensor([lane0 + 32 * (i // 16) + i % 16 for i in range(64)], device="cuda")
    err = (D[lanes] - ref).abs().max().item()
    assert err <= 1e-4 * ref.abs().max().item() + 1e-5, err
    other = torch.ones(128, dtype=torch.bool, device="cuda")
    other[lanes] = False
    assert (D[other] == 0).all()   # zeroed by the probe before the MMA, untouched by it
