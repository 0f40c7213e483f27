"""Build the ResNet-50 optimizer (no refresh), run 2 plain steps -- for ncu captures."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES
prec = sys.argv[1] if len(sys.argv) > 1 else "double"
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
g = torch.Generator(device=dev); g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
grads = [torch.randn(s, generator=g, device=dev) * 1e-2 for s in shapes]
# start_preconditioning_step=1 and frequency 1000: t=0,1 are plain steps; precondition runs at t=1 with
# (not ready) inverses masked -> use frequency=1 start=0 for a warm run instead when needed
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=1000,
                      start_preconditioning_step=0, precision=prec)
opt = P.Shampoo(params, cfg)
opt._ready_all = True
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    opt.step(grads)
torch.cuda.synchronize()
print("done")
