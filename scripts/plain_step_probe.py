"""One plain (non-refresh) ResNet-50 step bracketed by cudaProfilerStart/Stop, for ncu
(--profile-from-start off).  Steps 0..2 run first (t = 0 refresh), the profiled step is t = 3."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES[sys.argv[1] if len(sys.argv) > 1 else "resnet50"]]
g = torch.Generator(device=dev)
g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=50)
opt = P.Shampoo(params, cfg)
for t in range(4):
    grads = [torch.randn(s, generator=g, device=dev) * 1e-2 for s in shapes]
    torch.cuda.synchronize()
    if t == 3:
        torch.cuda.cudart().cudaProfilerStart()
    opt.step(grads)
    torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("ok")
