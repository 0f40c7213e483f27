"""Per-phase timing on the ResNet-50 set with CUDA events: refreshes (cold t=0, warm t=f, 2f) and plain steps."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

prec = sys.argv[1] if len(sys.argv) > 1 else "double"
freq = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
g = torch.Generator(device=dev); g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
grads = [[torch.randn(s, generator=g, device=dev) * 1e-2 for s in shapes] for _ in range(3)]
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=freq,
                      precision=prec)
opt = P.Shampoo(params, cfg)
lib = N.lib()
lib.shampoo_timing_enable(opt._ctx, 1)
names = ["stats", "root_inverse", "precondition", "graft_momentum", "apply"]
ms = (C.c_double * 5)(); cnt = (C.c_int64 * 5)()
for t in range(2 * freq + 1):
    opt.step(grads[t % 3])
    torch.cuda.synchronize()
    lib.shampoo_timing_get(opt._ctx, ms, cnt)
    if cnt[1]:
        print(f"t={t:3d} refresh {'cold' if t == 0 else 'warm'}: root_inverse {ms[1]:8.1f} ms")
lib.shampoo_timing_get(opt._ctx, None, None)
K = 10
for k in range(K):
    if opt.step_count % freq == 0:
        opt.advance_step()
    opt.step(grads[k % 3])
torch.cuda.synchronize()
lib.shampoo_timing_get(opt._ctx, ms, cnt)
sf, pf, n3 = C.c_double(), C.c_double(), C.c_double()
lib.shampoo_work(opt._ctx, C.byref(sf), C.byref(pf), C.byref(n3))
tot = 0.0
for i, n in enumerate(names):
    if i == 1:
        continue
    per = ms[i] / max(cnt[i], 1)
    tot += per
    extra = ""
    if n == "stats": extra = f"  ({sf.value/per/1e9:.1f} TF/s incl. prepare)"
    if n == "precondition": extra = f"  ({pf.value/per/1e9:.1f} TF/s incl. norms)"
    print(f"{n:16s} {per:8.3f} ms x{cnt[i]}{extra}")
print(f"plain step total {tot:.3f} ms")
