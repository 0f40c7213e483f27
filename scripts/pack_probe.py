"""One plain ResNet-50 step restricted to the parameters whose merged block order is argv[1]
("1", "2", "3" or "all"), bracketed by cudaProfilerStart/Stop for an ncu launch list: splits the
plain step's packing cost by operand layout (order-2 blocks: row + column packs of G; order-3
blocks: general two-index k maps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import planning
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

dev = torch.device("cuda:0")
which = sys.argv[1] if len(sys.argv) > 1 else "all"
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
if which != "all":
    shapes = [s for s in shapes if len(planning.merge_dims(s, 2048)) == int(which)]
print(which, len(shapes), sum(torch.Size(s).numel() for s in shapes))
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
