import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2309_06497_b200 as P
R = np.load('/root/repo/tests/golden/rootinv.npz')
cases = sorted({k.split("/")[0] for k in R.files})
for case in cases:
    a = R[f"{case}/a"]
    m = torch.as_tensor(a, device="cuda")
    for p in (2, 4, 6):
        for eps in (1e-12, 1e-6):
            (x,), st, it = P.batched_root_inverse([m], p, epsilon=eps)
            ref = R[f"{case}/eigh/p{p}/e{eps:g}"]
            x = x.cpu().numpy()
            print(case, p, eps, it[0], f"{np.linalg.norm(x-ref)/np.linalg.norm(ref):.2e}")
