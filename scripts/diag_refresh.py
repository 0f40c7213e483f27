"""Refresh diagnostics on the bench workload: per-factor-size Jacobi sweeps and time, cold vs warm.

Runs the ResNet-50 optimizer (bench config) to t=50, then re-solves the bias-corrected t=50 factors
cold with batched_root_inverse (grouped by root p) and prints sweeps per size plus wall time.
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

T = int(sys.argv[1]) if len(sys.argv) > 1 else 50
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
g = torch.Generator(device=dev); g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
g.manual_seed(1)
pool = [[torch.randn(s, generator=g, device=dev) * 1e-2 for s in shapes] for _ in range(T + 1)]  # fresh per step
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=50,
                      betas=(0.0, 0.999), epsilon=1e-12, momentum=0.9, use_nesterov=True, weight_decay=1e-4,
                      use_decoupled_weight_decay=True)
opt = P.Shampoo(params, cfg)
lib = N.lib()
lib.shampoo_timing_enable(opt._ctx, 1)
ms = (C.c_double * 5)(); cnt = (C.c_int64 * 5)()
for t in range(T + 1):
    lib.shampoo_timing_get(opt._ctx, None, None)
    opt.step(pool[t])
    torch.cuda.synchronize()
    lib.shampoo_timing_get(opt._ctx, ms, cnt)
    if cnt[1]:
        print(f"t={t}: optimizer refresh root_inverse {ms[1]:.1f} ms (stats {ms[0]:.2f} precond {ms[2]:.2f})", flush=True)
# cold re-solve of the current factors
corr = 1 - 0.999 ** (T + 1)
by_p = {}
for info in opt._blocks:
    if info.kind != N.BLOCK_SHAMPOO:
        continue
    for k in range(info.order):
        d = info.hi[k] - info.lo[k]
        f = opt._view(info.block_id, "factor", k).view(d, d).double() / corr
        by_p.setdefault(2 * info.order, []).append(f.clone())
tot = 0.0
for p, mats in sorted(by_p.items()):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    outs, status, sweeps = P.batched_root_inverse(mats, p, epsilon=1e-12)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    tot += dt
    hist = {}
    for m, s in zip(mats, sweeps):
        hist.setdefault(m.shape[0], []).append(s)
    def fmt(v):
        nw = [x - 100000 for x in v if x >= 100000]
        jb = [x for x in v if x < 100000]
        out = f"newton {len(nw)}" + (f" ({min(nw)}-{max(nw)} it)" if nw else "")
        if jb:
            out += f", jacobi {len(jb)} ({min(x % 1000 for x in jb)}-{max(x % 1000 for x in jb)} sw)"
        return out
    print(f"p={p}: {len(mats)} factors cold {dt*1e3:.1f} ms; solver by n: "
          + ", ".join(f"{n}:{fmt(v)}" for n, v in sorted(hist.items(), reverse=True)), flush=True)
print(f"cold total {tot*1e3:.1f} ms")
# per-size timing, one size at a time (cold)
for n in (2048, 1024, 512):
    mats = [m for p, ms_ in by_p.items() for m in ms_ if m.shape[0] == n]
    p_of = [p for p, ms_ in by_p.items() for m in ms_ if m.shape[0] == n]
    if not mats:
        continue
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    outs, status, sweeps = P.batched_root_inverse(mats[:1], p_of[0], epsilon=1e-12)
    torch.cuda.synchronize()
    print(f"single n={n}: {1e3*(time.perf_counter()-t0):.1f} ms sweeps={sweeps}", flush=True)
# accuracy of the cold re-solve against a float64 CPU eigh on a few factors
import numpy as np
for p, mats in sorted(by_p.items()):
    for m in mats[:3]:
        (x,), st, sw = P.batched_root_inverse([m], p, epsilon=1e-12)
        a = m.cpu().numpy()
        w, q = np.linalg.eigh(a)
        ref = (q * (w - min(w.min(), 0) + 1e-12) ** (-1.0 / p)) @ q.T
        xr = x.cpu().numpy()
        print(f"acc p={p} n={a.shape[0]} rel={np.linalg.norm(xr-ref)/np.linalg.norm(ref):.2e} sweeps={sw} "
              f"wmin={w.min():.2e} wmax={w.max():.2e}", flush=True)
