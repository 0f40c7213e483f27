"""Refresh cost over a longer run of the bench workload: fresh gradients every step (generated on the
device, never reused), prints the root-inverse phase time of every refresh (t = 0, f, 2f, ...)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

T = int(sys.argv[1]) if len(sys.argv) > 1 else 500
F = int(sys.argv[2]) if len(sys.argv) > 2 else 50
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
g = torch.Generator(device=dev); g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
g.manual_seed(1)
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=F,
                      betas=(0.0, 0.999), epsilon=1e-12, momentum=0.9, use_nesterov=True, weight_decay=1e-4,
                      use_decoupled_weight_decay=True)
opt = P.Shampoo(params, cfg)
lib = N.lib()
lib.shampoo_timing_enable(opt._ctx, 1)
ms = (C.c_double * 5)(); cnt = (C.c_int64 * 5)()
tot = 0.0
for t in range(T + 1):
    grads = [torch.randn(s, generator=g, device=dev) * 1e-2 for s in shapes]
    lib.shampoo_timing_get(opt._ctx, None, None)
    opt.step(grads)
    if t % F == 0:
        torch.cuda.synchronize()
        lib.shampoo_timing_get(opt._ctx, ms, cnt)
        tot += ms[1] if t else 0.0
        print(f"t={t:5d}: refresh root_inverse {ms[1]:8.1f} ms  guard {opt.guard_stats}", flush=True)
print(f"mean warm refresh {tot / max(T // F, 1):.1f} ms")
