"""Per-step timeline of the e2e pipeline (bench.py section 3): H2D / compute / snapshot / D2H spans
on their own streams, CUDA events relative to the window start, plain steps only (no refresh in
the window).  Diagnoses where the e2e step loses time against the device-only step."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
numels = [math.prod(s) for s in shapes]
n = sum(numels)
g = torch.Generator(device=dev); g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=1000,
                      betas=(0.0, 0.999), epsilon=1e-12, momentum=0.9, use_nesterov=True, weight_decay=1e-4,
                      use_decoupled_weight_decay=True)
mode = sys.argv[1] if len(sys.argv) > 1 else "deferred"
copies = sys.argv[2] if len(sys.argv) > 2 else "both"   # both | h2d | d2h | none
opt = P.Shampoo(params, cfg, check_finite="deferred" if mode == "deferred" else True)
K, NB = 12, 3
hg = [torch.randn(n).mul_(1e-2).pin_memory() for _ in range(K)]
hp = torch.empty(n).pin_memory()
df = [torch.empty(n, device=dev) for _ in range(NB)]
dg = [[v.view(s) for v, s in zip(torch.split(f, numels), shapes)] for f in df]
sf = [torch.empty(n, device=dev) for _ in range(2)]
sn = [[v.view(s) for v, s in zip(torch.split(f, numels), shapes)] for f in sf]
for k in range(3):
    df[0].copy_(hg[k]); opt.step(dg[0])
torch.cuda.synchronize()
st = torch.cuda.current_stream(); h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)
e0 = E()
spans = {k: {} for k in range(K)}
ev_in = [E() for _ in range(NB)]; ev_used = [E() for _ in range(NB)]
ev_snap = [E() for _ in range(2)]; ev_out = [E() for _ in range(2)]

def span(name, k, strm, fn):
    a, b = E(), E()
    a.record(strm); fn(); b.record(strm)
    spans[k][name] = (a, b)

def upload(k):
    b = k % NB
    with torch.cuda.stream(h2d):
        h2d.wait_event(e0)
        if k >= NB:
            h2d.wait_event(ev_used[b])
        if copies in ("both", "h2d"):
            span("h2d", k, h2d, lambda: df[b].copy_(hg[k], non_blocking=True))
        ev_in[b].record(h2d)

import time
e0.record(st)
t0 = time.perf_counter()
hostt = []
for k in range(NB - 1):
    upload(k)
for k in range(K):
    b, q = k % NB, k % 2
    if k + NB - 1 < K:
        upload(k + NB - 1)
    st.wait_event(ev_in[b])
    span("step", k, st, lambda: opt.step(dg[b]))
    ev_used[b].record(st)
    if k >= 2:
        st.wait_event(ev_out[q])
    span("snap", k, st, lambda: torch._foreach_copy_(sn[q], list(opt.params())))
    ev_snap[q].record(st)
    with torch.cuda.stream(d2h):
        d2h.wait_event(ev_snap[q])
        if copies in ("both", "d2h"):
            span("d2h", k, d2h, lambda: hp.copy_(sf[q], non_blocking=True))
        ev_out[q].record(d2h)
    hostt.append((time.perf_counter() - t0) * 1e3)
torch.cuda.synchronize()
steps = [spans[k]["step"] for k in range(3, K)]
print(f"mode {mode} copies {copies}: mean step span {sum(a.elapsed_time(b) for a, b in steps) / len(steps):.3f} ms")
print(f"mode {mode}; spans in ms from window start (start-end); host time at end of each iteration")
for k in range(K):
    row = " ".join(f"{nm} {e0.elapsed_time(a):7.2f}-{e0.elapsed_time(b):7.2f}" for nm, (a, b) in spans[k].items())
    print(f"step {k:2d}: {row}  host {hostt[k]:7.2f}")
