"""H2D / D2H throughput of the ResNet-50 parameter set (161 fp32 tensors, 102 MB) from pinned memory:
each direction alone and both concurrently on two streams (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
dev = torch.device("cuda:0")
hs = [torch.randn(s).pin_memory() for s in shapes]
hd = [torch.empty(s).pin_memory() for s in shapes]
ds = [torch.empty(s, device=dev) for s in shapes]
d2 = [torch.randn(s, device=dev) for s in shapes]
big_h = torch.randn(sum(t.numel() for t in hs)).pin_memory()
big_d = torch.empty_like(big_h, device=dev)
a, b = torch.cuda.Stream(), torch.cuda.Stream()
nb = 4 * sum(t.numel() for t in hs)
def run(h2d, d2h, big=False):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        if h2d:
            with torch.cuda.stream(a):
                if big: big_d.copy_(big_h, non_blocking=True)
                else:
                    for x, y in zip(ds, hs): x.copy_(y, non_blocking=True)
        if d2h:
            with torch.cuda.stream(b):
                for x, y in zip(hd, d2): x.copy_(y, non_blocking=True)
    torch.cuda.current_stream().wait_stream(a); torch.cuda.current_stream().wait_stream(b)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    return ms, nb / ms / 1e6
for name, args in [("h2d", (1, 0)), ("d2h", (0, 1)), ("both", (1, 1)), ("h2d one copy", (1, 0, True))]:
    ms, gbs = run(*args)
    print(f"{name:14s} {ms:6.2f} ms/step  {gbs:6.1f} GB/s per direction")
