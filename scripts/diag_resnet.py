"""Diagnostics: per-block direction error and per-factor root-inverse error on ResNet-50 block shapes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2309_06497_b200 as P
from oracle import shampoo_oracle as O

dev = torch.device("cuda:0")
shapes = [(2048, 512, 1, 1), (512, 512, 3, 3), (64, 3, 7, 7), (2048,), (1000, 2048), (256, 64, 1, 1),
          (128, 128, 3, 3), (1000,)]
eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-12
rng = np.random.default_rng(0)
params = [(rng.standard_normal(s) * 0.05).astype(np.float32) for s in shapes]
grng = np.random.default_rng(1)
grads = [[(grng.standard_normal(s) * 1e-2).astype(np.float32) for s in shapes] for _ in range(3)]
kw = dict(max_preconditioner_dim=2048, precondition_frequency=2, epsilon=eps)
cfg = P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, **kw)
oracle = O.OracleShampoo([p.astype(np.float64) for p in params], O.OracleConfig(grafting=O.GraftKind.ADAGRAD, **kw))
opt = P.Shampoo([torch.as_tensor(p, device=dev) for p in params], cfg)
for t in range(3):
    d_ref = oracle.step([g.astype(np.float64) for g in grads[t]])
    opt.step([torch.as_tensor(g, device=dev) for g in grads[t]])
    torch.cuda.synchronize()
    for (i, b), ref in d_ref.items():
        d = opt.direction(i, b).cpu().numpy()
        print(f"t={t} block ({i},{b}) shape={ref.shape} dir_rel={np.linalg.norm(d-ref)/np.linalg.norm(ref):.3e}")
    print("guard", opt.guard_stats)
tree = opt.state_tree()
for i, row in enumerate(oracle.states):
    for b, st in enumerate(row):
        for k, f in enumerate(st.factors):
            fg = tree["params"][i][b][f"factor{k}"]
            xg = tree["params"][i][b][f"inv_factor{k}"]
            xr = st.inverses[k]
            corr = 1 - 0.999 ** 3
            t0 = time.time()
            (x2,), status, sweeps = P.batched_root_inverse([torch.as_tensor(fg / corr, device=dev)], 2 * len(st.shape), epsilon=eps)
            torch.cuda.synchronize()
            dt = time.time() - t0
            x2 = x2.cpu().numpy()
            w = np.linalg.eigvalsh(fg / corr)
            print(f"factor ({i},{b},{k}) n={f.shape[0]} f_rel={np.linalg.norm(fg-f)/np.linalg.norm(f):.2e} "
                  f"inv_rel={np.linalg.norm(xg-xr)/np.linalg.norm(xr):.2e} re-solve rel={np.linalg.norm(x2-xr)/np.linalg.norm(xr):.2e} "
                  f"status={status} sweeps={sweeps} {dt*1e3:.1f}ms wmin={w.min():.3e} wmax={w.max():.3e}")
