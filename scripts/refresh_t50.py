"""Bench workload up to the t=50 refresh; the last step (the refresh) is bracketed by cuProfilerStart/Stop
(ncu --profile-from-start off captures only it)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
g = torch.Generator(device=dev); g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
g.manual_seed(1)
T = int(sys.argv[1]) if len(sys.argv) > 1 else 51
pool = [[torch.randn(s, generator=g, device=dev) * 1e-2 for s in shapes] for _ in range(T)]  # fresh per step
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=50,
                      betas=(0.0, 0.999), epsilon=1e-12, momentum=0.9, use_nesterov=True, weight_decay=1e-4,
                      use_decoupled_weight_decay=True)
opt = P.Shampoo(params, cfg)
for t in range(T):
    if t == T - 1:
        torch.cuda.synchronize()
        ctypes.CDLL("libcuda.so.1").cuProfilerStart()
    opt.step(pool[t])
torch.cuda.synchronize()
ctypes.CDLL("libcuda.so.1").cuProfilerStop()
print("done", opt.guard_stats)
