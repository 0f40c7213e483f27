"""Factor-statistics slice count vs accuracy (ResNet-50, b=2048, f=50, eps=1e-12).

Two optimizer contexts fed identical gradients: the FP64-class default (8 slices, pinned to the oracle by
the parity tests) and SHAMPOO_STATS_SLICES=k.  Full steps from t = 0 (rank-deficient factors, low-rank
refreshes) to t = T1, then statistics-only fast-forward to T0 - 50 and one full precondition cycle
(steady state).  Reports per refresh window the worst per-block relative Frobenius error of factors,
inverses and directions, and the stats phase ms of both.

    python scripts/stats_slices_probe.py [T1] [T0] [k ...]
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

T1 = int(sys.argv[1]) if len(sys.argv) > 1 else 151
T0 = int(sys.argv[2]) if len(sys.argv) > 2 else 2600
KS = [int(x) for x in sys.argv[3:]] or [6]
EPS = float(os.environ.get("PROBE_EPS", "1e-12"))
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
numels = [math.prod(s) for s in shapes]
n = sum(numels)
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=50,
                      epsilon=EPS, momentum=0.9, use_nesterov=True, weight_decay=1e-4)


def make(k):
    if k == 8:
        os.environ.pop("SHAMPOO_STATS_SLICES", None)
    else:
        os.environ["SHAMPOO_STATS_SLICES"] = str(k)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
    return P.Shampoo(params, cfg), params


def rel(a, b):
    nb = float(torch.linalg.vector_norm(b))
    return float(torch.linalg.vector_norm(a - b)) / nb if nb > 0 else float(torch.linalg.vector_norm(a))


def compare(o8, ok, tag):
    worst = {"factor": 0.0, "inv_factor": 0.0, "direction": 0.0}
    for info in o8._blocks:
        shape = tuple(info.hi[k] - info.lo[k] for k in range(info.order))
        d8 = o8.direction(info.param_index, info.block_index).double()
        dk = ok.direction(info.param_index, info.block_index).double()
        worst["direction"] = max(worst["direction"], rel(dk, d8))
        if info.kind != N.BLOCK_SHAMPOO:
            continue
        for m in range(info.order):
            for name in ("factor", "inv_factor"):
                a, b = o8._view(info.block_id, name, m), ok._view(info.block_id, name, m)
                if a is not None and b is not None:
                    worst[name] = max(worst[name], rel(b.double(), a.double()))
    print(f"{tag}: worst rel factor {worst['factor']:.2e} inverse {worst['inv_factor']:.2e} "
          f"direction {worst['direction']:.2e}", flush=True)


lib = N.lib()
for k in KS:
    (o8, p8), (ok, pk) = make(8), make(k)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    flat = torch.empty(n, device=dev)

    def grads():
        torch.randn(n, generator=gen, device=dev, out=flat)
        flat.mul_(1e-2)
        return [v.view(sh) for v, sh in zip(torch.split(flat, numels), shapes)]

    while o8.step_count < T1:
        g = grads()
        o8.step(g)
        ok.step(g)
        t = o8.step_count - 1
        if t % 50 in (0, 1, 49):
            compare(o8, ok, f"S={k} t={t}")
    s = torch.cuda.current_stream().cuda_stream
    while o8.step_count < T0 - 50:
        g = grads()
        gp = N.ptr_array([x.data_ptr() for x in g])
        for opt, params in ((o8, p8), (ok, pk)):
            pp = N.ptr_array([p.data_ptr() for p in params])
            N.check(lib.shampoo_stats_update(opt._ctx, gp, pp, N.DTYPE_F32, opt.step_count, s))
            opt.advance_step()
    while o8.step_count <= T0 + 1:
        g = grads()
        o8.step(g)
        ok.step(g)
        t = o8.step_count - 1
        if t % 50 in (0, 1, 49):
            compare(o8, ok, f"S={k} t={t} (steady)")
    for opt, tag in ((o8, "S=8"), (ok, f"S={k}")):
        lib.shampoo_timing_enable(opt._ctx, 1)
        import ctypes as C
        lib.shampoo_timing_get(opt._ctx, None, None)
        for _ in range(5):
            opt.step(grads())
        ms = (C.c_double * 5)()
        cnt = (C.c_int64 * 5)()
        lib.shampoo_timing_get(opt._ctx, ms, cnt)
        lib.shampoo_timing_enable(opt._ctx, 0)
        print(f"{tag}: stats {ms[0] / max(cnt[0], 1):.3f} ms/step", flush=True)
    del o8, ok
