"""e2e pipeline around a steady-state refresh step: per-step CUDA-event times with the H2D / D2H
copies on (bench.py section 3) or off, so the cost the copies add to a refresh step can be seen.

    python scripts/e2e_refresh_probe.py [T0] [copies: none|h2d|d2h|both]
"""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

T0 = int(sys.argv[1]) if len(sys.argv) > 1 else 2600
copies = sys.argv[2] if len(sys.argv) > 2 else "both"
dev = torch.device("cuda:0")
shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
numels = [math.prod(s) for s in shapes]
n = sum(numels)
g = torch.Generator(device=dev); g.manual_seed(0)
params = [torch.randn(s, generator=g, device=dev) * 0.05 for s in shapes]
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, max_preconditioner_dim=2048, precondition_frequency=50,
                      betas=(0.0, 0.999), epsilon=1e-12, momentum=0.9, use_nesterov=True, weight_decay=1e-4,
                      use_decoupled_weight_decay=True)
opt = P.Shampoo(params, cfg, check_finite="deferred")
flat = torch.empty(n, device=dev)
def fresh():
    torch.randn(n, generator=g, device=dev, out=flat); flat.mul_(1e-2)
    return [v.view(s) for v, s in zip(torch.split(flat, numels), shapes)]
lib = N.lib(); st = torch.cuda.current_stream()
pp = N.ptr_array([p.data_ptr() for p in params])
while opt.step_count < T0 - 50:
    gg = fresh(); gp = N.ptr_array([x.data_ptr() for x in gg])
    N.check(lib.shampoo_stats_update(opt._ctx, gp, pp, N.DTYPE_F32, opt.step_count, st.cuda_stream)); opt.advance_step()
while opt.step_count < T0:
    opt.step(fresh())
torch.cuda.synchronize()
K, NB = 6, 3
hg = [torch.randn(n).mul_(1e-2).pin_memory() for _ in range(K)]
hp = torch.empty(n).pin_memory()
df = [torch.empty(n, device=dev) for _ in range(NB)]
dg = [[v.view(s) for v, s in zip(torch.split(f, numels), shapes)] for f in df]
sf = [torch.empty(n, device=dev) for _ in range(2)]
sn = [[v.view(s) for v, s in zip(torch.split(f, numels), shapes)] for f in sf]
for b in range(NB):
    df[b].copy_(hg[b % K])
if os.environ.get("PROBE_WARM", "1") == "1":  # first-use costs outside the window (bench.py does the same)
    for q in range(2):
        torch._foreach_copy_(sn[q], list(opt.params()))
        hp.copy_(sf[q], non_blocking=True)
h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)
ev = [E() for _ in range(K + 1)]
ev_in = [E() for _ in range(NB)]; ev_used = [E() for _ in range(NB)]
ev_snap = [E() for _ in range(2)]; ev_out = [E() for _ in range(2)]
torch.cuda.synchronize()
ev[0].record(st)
def upload(k):
    b = k % NB
    with torch.cuda.stream(h2d):
        h2d.wait_event(ev[0])
        if k >= NB:
            h2d.wait_event(ev_used[b])
        if copies in ("both", "h2d"):
            df[b].copy_(hg[k], non_blocking=True)
        ev_in[b].record(h2d)
for k in range(NB - 1):
    upload(k)
for k in range(K):
    b, q = k % NB, k % 2
    if k + NB - 1 < K:
        upload(k + NB - 1)
    st.wait_event(ev_in[b])
    opt.step(dg[b])
    ev_used[b].record(st)
    if k >= 2:
        st.wait_event(ev_out[q])
    torch._foreach_copy_(sn[q], list(opt.params()))
    ev_snap[q].record(st)
    with torch.cuda.stream(d2h):
        d2h.wait_event(ev_snap[q])
        if copies in ("both", "d2h"):
            hp.copy_(sf[q], non_blocking=True)
        ev_out[q].record(d2h)
    ev[k + 1].record(st)
torch.cuda.synchronize()
print(f"copies {copies}: per-step ms (step 0 = refresh)",
      [round(ev[k].elapsed_time(ev[k + 1]), 2) for k in range(K)])

# the same optimizer, resident gradients, straight to the next refresh: is the refresh itself slower
# inside the e2e loop, or is the difference the loop?
while opt.step_count % 50 != 0:
    opt.step(fresh())
torch.cuda.synchronize()
e0, e1 = E(), E()
gg = fresh()
e0.record(st)
opt.step(gg)
e1.record(st)
torch.cuda.synchronize()
print(f"next refresh (t={opt.step_count - 1}) with resident gradients: {e0.elapsed_time(e1):.2f} ms")
