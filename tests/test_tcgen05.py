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


@pytest.mark.parametrize("precision", ["double", "single"])
@pytest.mark.parametrize("beta1", [0.0, 0.9])
def test_dual_pack_bitwise_equal_to_per_operand_packs(cuda_device, monkeypatch, precision, beta1):
    """Transposed operand pairs (a block's row and column statistics, a mode-0 statistic and the
    first mode product's B operand) packed by k_oz_dual_exp + k_oz_pack_dual write the same slice
    bytes and exponents as the per-operand k_oz_rowexp + k_oz_pack passes: bit-identical steps.
    Ragged shapes cover partial tiles (rows/columns not multiples of 64/32) and order-3 blocks."""
    import torch

    shapes = [(37, 100), (100, 37), (64, 64), (130, 65, 3), (40, 40, 40), (33, 70, 45), (5, 7, 3), (300, 2),
              (1, 50), (513, 129)]
    rng = np.random.default_rng(5)
    init = [rng.standard_normal(s) * 0.1 for s in shapes]
    grads = [[rng.standard_normal(s) * 10.0 ** rng.integers(-3, 2) for s in shapes] for _ in range(4)]
    dt = torch.float64 if precision == "double" else torch.float32

    def run(dual: bool):
        monkeypatch.setenv("SHAMPOO_OZ_DUAL_PACK", "1" if dual else "0")
        cfg = P.ShampooConfig(lr=0.05, betas=(beta1, 0.999), max_preconditioner_dim=128, precondition_frequency=2,
                              grafting=P.GraftKind.ADAGRAD, precision=precision)
        opt = P.Shampoo([torch.as_tensor(x, device=cuda_device, dtype=dt) for x in init], cfg)
        for g in grads:
            opt.step([torch.as_tensor(x, device=cuda_device, dtype=dt) for x in g])
        torch.cuda.synchronize()
        return [p.cpu().numpy() for p in opt.params()]

    got, ref = run(True), run(False)
    monkeypatch.delenv("SHAMPOO_OZ_DUAL_PACK")
    for a, b in zip(got, ref):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_tc_gemm_special_values(cuda_device, dtype):
    """Slicing edge cases: signed zeros, subnormals, exact powers of two (the row maximum sits on
    the exponent boundary), all-zero rows, magnitudes spread over 2^-90 .. 2^40 within one row, and
    ties of the last digit -- against the FP64 product within the Ozaki bound."""
    import torch

    dt = getattr(torch, dtype)
    g = torch.Generator(device=cuda_device).manual_seed(11)
    m, n, k = 70, 45, 300
    a = torch.randn(m, k, device=cuda_device, generator=g, dtype=torch.float64)
    a *= torch.exp2(torch.randint(-90, 41, (m, k), device=cuda_device, generator=g).double())
    a[0] = 0.0
    a[1] = -0.0
    a[2, :10] = 2.0 ** torch.arange(10, device=cuda_device, dtype=torch.float64)  # exact powers of two
    a[3, ::2] = -(2.0 ** 20)
    a[3, 1::2] = 2.0 ** -30 * (1 + 2.0 ** -40)
    tiny = 5e-324 if dtype == "float64" else 1e-45
    a[4, :] = tiny
    a[4, 0] = 1.0
    a[5, :] = 1.0 + 2.0 ** -45
    a[6, :] = 1.0 + 2.0 ** -35  # 0.5 + 2^-36 after scaling: a remainder of exactly half a unit at S = 5
    b = torch.randn(n, k, device=cuda_device, generator=g, dtype=torch.float64)
    b[7] = -b[7]
    a, b = a.to(dt), b.to(dt)
    c = P.tc_gemm(a, b, torch.zeros(m, n, device=cuda_device, dtype=dt))
    torch.cuda.synchronize()
    ref = a.double() @ b.double().T
    # Ozaki bound in units of the row scales 2^ea 2^eb (the rows here span 130 binades, so the
    # |a||b|-relative bound of the dense tests does not apply): each operand is truncated to
    # 2^-7S of its row scale and the dropped slice products are below S 2^-7S, per term of k
    S = 8 if dtype == "float64" else 5
    ea = torch.frexp(a.double().abs().amax(1)).exponent.double()
    eb = torch.frexp(b.double().abs().amax(1)).exponent.double()
    unit = torch.exp2(ea[:, None] + eb[None, :] - 7 * S)
    out_round = (6e-8 if dtype == "float32" else 1.2e-16) * ref.abs()
    excess = (c.double() - ref).abs() - (2 * (S + 2) * k * unit + out_round)
    assert excess.max().item() <= 0, excess.max().item()
    assert torch.all(c[:2] == 0)
