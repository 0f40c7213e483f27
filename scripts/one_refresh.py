"""Run the ResNet-50 optimizer through one cold refresh (t=0) and one warm refresh (t=2) -- for ncu."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
g = torch.Generator(device=dev); g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
grads = [[torch.randn(s, generator=g, device=dev) * 1e-2 for s in shapes] for _ in range(2)]
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=2)
opt = P.Shampoo(params, cfg)
for t in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    opt.step(grads[t % 2])
torch.cuda.synchronize()
print("done", opt.guard_stats)
