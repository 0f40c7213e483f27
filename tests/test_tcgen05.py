"""tcgen05 int8 tensor-core GEMM with Ozaki splitting (exact int32 accumulation, slice diagonals
combined in FP64) against an FP64 torch reference: the engine behind the factor statistics and
the mode products (precond.py:161-174) of both precisions."""

import numpy as np
import pytest

import paper_2309_06497_b200 as P

pytestmark = pytest.mark.gpu

# error per entry relative to sum_k |a_ik||b_jk| (the DGEMM-style bound); the Ozaki split bounds it
# by ~2 * 2^(-7 S) * max|a_i.| max|b_j.| / mean(|a||b|): 8 slices (double), 5 slices (single)
TOL = {"float64": 1e-14, "float32": 2e-7}


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("m,n,k", [(128, 64, 32), (200, 100, 70), (1, 1, 1), (3, 5, 7), (512, 384, 1000),
                                   (130, 260, 9000)])
def test_tc_gemm_matches_fp64(cuda_device, dtype, m, n, k):
    import torch

    dt = getattr(torch, dtype)
    g = torch.Generator(device=cuda_device).manual_seed(m * 7 + n * 3 + k)
    a = torch.randn(m, k, device=cuda_device, generator=g, dtype=torch.float64)
    b = torch.randn(n, k, device=cuda_device, generator=g, dtype=torch.float64) * 1e-3
    c0 = torch.randn(m, n, device=cuda_device, generator=g, dtype=torch.float64)
    a, b, c0 = a.to(dt), b.to(dt), c0.to(dt)
    c = P.tc_gemm(a, b, c0.clone(), alpha=0.5, beta=2.0)
    torch.cuda.synchronize()
    ref = 0.5 * (a.double() @ b.double().T) + 2.0 * c0.double()
    scale = 0.5 * (a.double().abs() @ b.double().abs().T) + 2.0 * c0.double().abs()
    out_round = 6e-8 if dtype == "float32" else 1.2e-16
    err = ((c.double() - ref).abs() / scale).max().item()
    assert err <= TOL[dtype] + out_round, err


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("n,k", [(64, 512), (300, 4096), (1000, 50), (3, 20000)])
def test_tc_syrk_symmetric_ema(cuda_device, dtype, n, k):
    """Factor EMA F <- beta F + (1 - beta) X X^T: exactly symmetric, and no accumulation bias
    (fp32 tensor-core accumulation is biased by ~K/8 ulp: 3e-5 at K = 4096)."""
    import torch

    dt = getattr(torch, dtype)
    g = torch.Generator(device=cuda_device).manual_seed(n + k)
    x = (torch.randn(n, k, device=cuda_device, generator=g, dtype=torch.float64) * 1e-2).to(dt)
    f0 = (x[:, :8].double() @ x[:, :8].double().T).to(dt)
    f = P.tc_gemm(x, x, f0.clone(), symmetric=True, alpha=1 - 0.999, beta=0.999)
    torch.cuda.synchronize()
    assert torch.equal(f, f.T)  # mirrored tiles: exactly symmetric (precond.py:165)
    ref = 0.001 * (x.double() @ x.double().T) + 0.999 * f0.double()
    rel = ((f.double() - ref).norm() / ref.norm()).item()
    assert rel <= (1e-15 if dtype == "float64" else 1e-7), rel


def test_tc_gram_of_rank_deficient_stays_psd(cuda_device):
    """X X^T of a rank-r X computed from the truncated slices is the exact Gram of a perturbed X:
    its null space eigenvalues stay at FP64 rounding level (eps = 1e-12 parity, matfun.py:148)."""
    import torch

    g = torch.Generator(device=cuda_device).manual_seed(5)
    x = torch.randn(256, 40, device=cuda_device, generator=g, dtype=torch.float64) * 1e-2
    f = P.tc_gemm(x, x, symmetric=True)
    w = torch.linalg.eigvalsh(f).cpu().numpy()
    assert w[:216].max() <= 1e-16 * w.max() * 256 and w[:216].min() >= -1e-16 * w.max() * 256


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("m,n,k,sym", [(200, 100, 70, False), (512, 384, 1000, False), (300, 300, 4096, True),
                                       (130, 260, 9000, False)])
def test_tma_and_bulk_copy_paths_bitwise_equal(cuda_device, monkeypatch, dtype, m, n, k, sym):
    """The TMA tensor-map loads (cores past the operand's end zero-filled) and the per-slice bulk
    copies feed identical tiles: bit-identical results, including split-K (k = 9000) and SYRK."""
    import torch

    dt = getattr(torch, dtype)
    g = torch.Generator(device=cuda_device).manual_seed(m + 11 * n + k)
    a = torch.randn(m, k, device=cuda_device, generator=g, dtype=torch.float64).to(dt)
    b = a if sym else torch.randn(n, k, device=cuda_device, generator=g, dtype=torch.float64).to(dt)
    c0 = torch.randn(m, n, device=cuda_device, generator=g, dtype=torch.float64).to(dt)
    if sym:
        c0 = (c0 + c0.T) / 2
    monkeypatch.delenv("SHAMPOO_OZ_NO_TMA", raising=False)
    c_tma = P.tc_gemm(a, b, c0.clone(), symmetric=sym, alpha=0.5, beta=2.0)
    monkeypatch.setenv("SHAMPOO_OZ_NO_TMA", "1")
    c_blk = P.tc_gemm(a, b, c0.clone(), symmetric=sym, alpha=0.5, beta=2.0)
    torch.cuda.synchronize()
    assert torch.equal(c_tma, c_blk)
