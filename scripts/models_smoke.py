"""Every model shape set of SURVEY §8d through a refresh-heavy run (f=10, 31 steps, fresh gradients):
per-refresh time, guard counters, finite parameters.  `python scripts/models_smoke.py [precision]`."""
import ctypes as C, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES
prec = sys.argv[1] if len(sys.argv) > 1 else "double"
dev = torch.device("cuda:0")
for name, shapes in MODEL_SHAPES.items():
    shapes = [tuple(s) for s in shapes]
    g = torch.Generator(device=dev); g.manual_seed(0)
    params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
    bdim = 2048 if name == "resnet50" else (512 if name == "mlp" else 1024)
    graft = P.GraftKind.ADAGRAD if name in ("resnet50", "mlp") else P.GraftKind.ADAM
    cfg = P.ShampooConfig(grafting=graft, max_preconditioner_dim=bdim, precondition_frequency=10, epsilon=1e-12,
                          momentum=0.9, use_nesterov=True, precision=prec)
    opt = P.Shampoo(params, cfg)
    lib = N.lib(); lib.shampoo_timing_enable(opt._ctx, 1)
    ms = (C.c_double * 5)(); cnt = (C.c_int64 * 5)()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for t in range(31):
        opt.step([torch.randn(s, generator=g, device=dev) * 1e-2 for s in shapes])
    torch.cuda.synchronize(); wall = time.perf_counter() - t0
    lib.shampoo_timing_get(opt._ctx, ms, cnt)
    finite = all(torch.isfinite(p).all().item() for p in opt.params())
    print(f"{name:14s} {len(shapes):4d} tensors {sum(math.prod(s) for s in shapes)/1e6:7.1f}M params: "
          f"refresh {ms[1]/max(cnt[1],1):7.1f} ms x{cnt[1]}, plain phases {(ms[0]+ms[2]+ms[3]+ms[4])/31:6.2f} ms/step, "
          f"wall {wall:5.1f} s, finite {finite}, guard {opt.guard_stats}", flush=True)
    del opt, params
    torch.cuda.empty_cache()
