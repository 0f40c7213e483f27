"""Steady-state refresh probe: synthetic factors shaped like the ResNet-50 blocks at step T (EMA of
fresh N(0, 0.01^2) gradients, beta2 = 0.999, bias-corrected), solved by batched_root_inverse grouped by
root p.  Vector blocks (order 1) get the exact rank-T EMA Gram; order-2 blocks a Gram of
min(T K, 6 d) Gaussian columns (same conditioning class).  cudaProfilerStart brackets the solves
(ncu --profile-from-start off)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import math
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2250
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
params = [torch.zeros(s, device=dev) for s in shapes]
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=50,
                      epsilon=1e-12)
opt = P.Shampoo(params, cfg)
g = torch.Generator(device=dev); g.manual_seed(3)
beta, corr = 0.999, 1 - 0.999 ** (T + 1)
by_p = {}
for info in opt._blocks:
    if info.kind != N.BLOCK_SHAMPOO:
        continue
    dims = [info.hi[k] - info.lo[k] for k in range(info.order)]
    numel = math.prod(dims)
    for k, d in enumerate(dims):
        K = numel // d
        if info.order == 1:
            w = ((1 - beta) * beta ** torch.arange(T, -1, -1, device=dev, dtype=torch.float64)).sqrt()
            G = torch.randn(d, T + 1, generator=g, device=dev, dtype=torch.float64) * 1e-2 * w
            A = G @ G.T / corr
        else:
            cols = min((T + 1) * K, 6 * d)
            G = torch.randn(d, cols, generator=g, device=dev, dtype=torch.float64) * 1e-2
            A = G @ G.T * (K / cols)  # bias-corrected EMA of K-column Grams: E[A] = K 1e-4 I
        by_p.setdefault(2 * info.order, []).append(A)
del opt
torch.cuda.synchronize()
for rep in range(2):
    if rep == 1:
        torch.cuda.cudart().cudaProfilerStart()
    tot = 0.0
    for p, mats in sorted(by_p.items()):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        outs, status, its = P.batched_root_inverse(mats, p, epsilon=1e-12)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        tot += dt
        hist = {}
        for m, s in zip(mats, its):
            hist.setdefault(m.shape[0], []).append(f"N{s - 100000}" if s >= 100000 else f"j{s % 1000}")
        print(f"rep {rep} p={p}: {len(mats)} factors {dt*1e3:.1f} ms; " +
              " ".join(f"{n}:{','.join(v)}" for n, v in sorted(hist.items(), reverse=True)), flush=True)
    print(f"rep {rep} total {tot*1e3:.1f} ms", flush=True)
torch.cuda.cudart().cudaProfilerStop()
