"""Quick per-phase timing of plain (non-refresh) steps on the ResNet-50 set (no refresh in window)."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

prec = sys.argv[1] if len(sys.argv) > 1 else "double"
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
g = torch.Generator(device=dev); g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
grads = [[torch.randn(s, generator=g, device=dev) * 1e-2 for s in shapes] for _ in range(2)]
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=1000,
                      start_preconditioning_step=0, precision=prec)
opt = P.Shampoo(params, cfg)
lib = N.lib()
t0 = time.time()
opt.step(grads[0])  # t=0 refresh (cold)
torch.cuda.synchronize()
print(f"refresh step (cold, t=0): {1e3*(time.time()-t0):.1f} ms wall")
for k in range(3):
    opt.step(grads[k % 2])
torch.cuda.synchronize()
lib.shampoo_timing_enable(opt._ctx, 1)
lib.shampoo_timing_get(opt._ctx, None, None)
K = 10
for k in range(K):
    opt.step(grads[k % 2])
torch.cuda.synchronize()
ms = (C.c_double * 5)(); cnt = (C.c_int64 * 5)()
lib.shampoo_timing_get(opt._ctx, ms, cnt)
sf, pf, n3 = C.c_double(), C.c_double(), C.c_double()
lib.shampoo_work(opt._ctx, C.byref(sf), C.byref(pf), C.byref(n3))
names = ["stats", "root_inverse", "precondition", "graft_momentum", "apply"]
for i, n in enumerate(names):
    per = ms[i] / max(cnt[i], 1)
    extra = ""
    if n == "stats": extra = f"  ({sf.value/per/1e9:.1f} TF/s incl. prepare)"
    if n == "precondition": extra = f"  ({pf.value/per/1e9:.1f} TF/s incl. norms)"
    print(f"{n:16s} {per:8.3f} ms x{cnt[i]}{extra}")
print("plain step total", sum(ms[i] / max(cnt[i], 1) for i in (0, 2, 3, 4)), "ms")
