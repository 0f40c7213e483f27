"""Mode-product slice count vs accuracy at the steady state (ResNet-50, b=2048, f=50, eps=1e-12).

Two optimizer contexts fed identical gradients: one with the default 8 slices (FP64 class, pinned to
the oracle by tests/test_gpu_parity.py), one with SHAMPOO_PREC_SLICES=k.  Factors and inverses are
identical (they do not depend on the mode products); the directions differ by the truncation of the
mode-product operands only.  Reports the worst per-block relative Frobenius error of the directions
on a refresh step and the stale steps after it, and the precondition phase ms of each context.

    python scripts/slices_probe.py [T0] [k ...]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

T0 = int(sys.argv[1]) if len(sys.argv) > 1 else 2600
KS = [int(x) for x in sys.argv[2:]] or [3, 4, 5, 6]
EPS = float(os.environ.get("PROBE_EPS", "1e-12"))
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
numels = [math.prod(s) for s in shapes]
n = sum(numels)
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=50,
                      epsilon=EPS)


def make(k):
    os.environ["SHAMPOO_PREC_SLICES"] = str(k)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
    return P.Shampoo(params, cfg), params


lib = N.lib()
for k in KS:
    opts = [make(8), make(k)]
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    flat = torch.empty(n, device=dev)
    s = torch.cuda.current_stream().cuda_stream

    def grads():
        torch.randn(n, generator=gen, device=dev, out=flat)
        flat.mul_(1e-2)
        return [v.view(sh) for v, sh in zip(torch.split(flat, numels), shapes)]

    while opts[0][0].step_count < T0 - 50:
        g = grads()
        gp = N.ptr_array([x.data_ptr() for x in g])
        for opt, params in opts:
            pp = N.ptr_array([p.data_ptr() for p in params])
            N.check(lib.shampoo_stats_update(opt._ctx, gp, pp, N.DTYPE_F32, opt.step_count, s))
            opt.advance_step()
    worst = {}
    for t in range(T0 - 50, T0 + 4):
        g = grads()
        for opt, _ in opts:
            opt.step(g)
        if t >= T0:
            torch.cuda.synchronize()
            w = 0.0
            for b in opts[0][0]._blocks:
                a = opts[0][0].direction(b.param_index, b.block_index)
                c = opts[1][0].direction(b.param_index, b.block_index)
                w = max(w, float((c - a).norm() / a.norm().clamp_min(1e-300)))
            worst[t] = w
    # precondition phase timing of both contexts (one plain step each)
    ms = []
    for opt, _ in opts:
        lib.shampoo_timing_enable(opt._ctx, 1)
        lib.shampoo_timing_get(opt._ctx, None, None)
        for _ in range(5):
            opt.step(grads())
        m = (N.C.c_double * 5)() if hasattr(N, "C") else None
        import ctypes as C
        m = (C.c_double * 5)()
        c = (C.c_int64 * 5)()
        lib.shampoo_timing_get(opt._ctx, m, c)
        lib.shampoo_timing_enable(opt._ctx, 0)
        ms.append(m[2] / max(c[2], 1))
    print(f"eps={EPS:g} S={k}: worst per-block direction rel err vs S=8 " +
          " ".join(f"t={t}:{w:.2e}" for t, w in worst.items()) +
          f" | precondition ms S=8 {ms[0]:.3f}, S={k} {ms[1]:.3f}", flush=True)
    del opts
    torch.cuda.empty_cache()
