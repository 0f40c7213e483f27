"""Steady-state parity (VERDICT r1 "what's weak" #1): the refresh routes the bench takes after
thousands of steps, against the float64 oracle.

Every distinct ResNet-50 block shape at b=2048 (28 shapes, factor dims 7..2048, orders 1/2/3, root
p = 2/4/6) gets oracle-built steady-state factors -- vector factors the exact EMA Gram of T = 2600
fresh gradients (beta2 = 0.999, full rank, ill-conditioned like the bench's), matrix factors Grams
of 4 d Gaussian columns -- loaded into both the oracle and the device optimizer (load_state_tree),
then two steps run on both: a refresh step t0 (a multiple of f) and a stale step t0 + 1.  Each
solver route is forced in turn through the context's environment switches (read at context
creation): the default scaled coupled-Newton pre-pass, unscaled Newton (SHAMPOO_NEWTON_SCALE=0), the
FP64 block-Jacobi eigensolver (SHAMPOO_EIG_NEWTON=0), and the low-rank range compression (early
state: vector factors of structural rank 100 < d).  A 2-step run over all 161 ResNet-50 tensors
from t = 0 covers the rank-deficient start.

Tolerances (written per assert): directions <= 1e-3 relative Frobenius per block (north_star);
inverse factors <= 1e-7 where the request is well posed (eps dominates the float64 eigenvalue noise
of any backward-stable solver), else the direction bound only; all routes agree with each other to
the same bounds; guard counters equal.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

import paper_2309_06497_b200 as P
from oracle import shampoo_oracle as O
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES

pytestmark = pytest.mark.gpu

F = 50
T0 = 2600
BETA2 = 0.999


def rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


def block_shapes():
    blocks = O.enumerate_blocks(MODEL_SHAPES["resnet50"], 2048)
    seen = []
    for b in blocks:
        if b.shape not in seen:
            seen.append(b.shape)
    return seen


def steady_factor(rng, d: int, k_cols: int, steps: int) -> np.ndarray:
    """Bias-uncorrected EMA factor after `steps` steps of N(0, 1e-4) gradients with k_cols columns
    per step (the mode's other dims): vector blocks exactly (d x steps weighted Gram), matrix blocks
    as a Gram of min(steps k_cols, 4 d) columns with the EMA's total weight."""
    if k_cols == 1:
        w = np.sqrt((1 - BETA2) * BETA2 ** np.arange(steps - 1, -1, -1))
        z = rng.standard_normal((d, steps)) * 1e-2 * w
    else:
        m = min(steps * k_cols, 4 * d)
        z = rng.standard_normal((d, m)) * 1e-2 * math.sqrt((1 - BETA2 ** steps) * k_cols / m)
    a = z @ z.T
    return (a + a.T) / 2


def build_state(shapes, eps, steps, seed=0, momentum_scale=1e-3):
    """Oracle optimizer at step t0 with steady-state factors, graft accumulators and momentum; the
    matching device state tree."""
    rng = np.random.default_rng(seed)
    params = [(rng.standard_normal(s) * 0.05).astype(np.float32).astype(np.float64) for s in shapes]
    cfg = dict(max_preconditioner_dim=2048, precondition_frequency=F, epsilon=eps, betas=(0.0, BETA2))
    ocfg = O.OracleConfig(grafting=O.GraftKind.ADAGRAD, **cfg)
    oracle = O.OracleShampoo([p.copy() for p in params], ocfg)  # the oracle updates its arrays in place
    t0 = int(math.ceil(steps / F)) * F
    oracle.t = t0
    tree = {"t": t0, "params": {}}
    for i, row in enumerate(oracle.states):
        tree["params"][i] = {}
        for b, st in enumerate(row):
            n = math.prod(st.shape)
            st.graft_step = steps
            st.graft_acc = rng.chisquare(steps, size=st.shape) * 1e-4
            st.momentum = rng.standard_normal(st.shape) * momentum_scale
            entry = {"kind": st.kind, "graft_step": steps, "graft_accumulator": st.graft_acc.copy(),
                     "momentum": st.momentum.copy()}
            if st.kind == "shampoo":
                st.step = steps
                st.last_inverse_step = -1
                st.factors = [steady_factor(rng, d, n // d, steps) for d in st.shape]
                st.inverses = None
                entry.update(step=steps, last_inverse_step=-1)
                for k, f in enumerate(st.factors):
                    entry[f"factor{k}"] = f.copy()
            tree["params"][i][b] = entry
    return params, oracle, tree, P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, **cfg)


def grads_for(shapes, seed, count):
    rng = np.random.default_rng(seed)
    return [[(rng.standard_normal(s) * 1e-2).astype(np.float32).astype(np.float64) for s in shapes]
            for _ in range(count)]


_ORACLE_CACHE: dict = {}


def oracle_run(key, shapes, eps, steps, **kw):
    """Oracle directions and inverses of the two steps (cached per (key, eps))."""
    if (key, eps) not in _ORACLE_CACHE:
        params, oracle, tree, cfg = build_state(shapes, eps, steps, **kw)
        dirs = [oracle.step(g) for g in grads_for(shapes, 1, 2)]
        inv = {(i, b): [x.copy() for x in st.inverses] for i, row in enumerate(oracle.states)
               for b, st in enumerate(row) if st.kind == "shampoo"}
        _ORACLE_CACHE[(key, eps)] = (params, tree, cfg, dirs, inv,
                                     (oracle.guard.primary, oracle.guard.double_retry,
                                      oracle.guard.fallback_previous, oracle.guard.fallback_identity))
    return _ORACLE_CACHE[(key, eps)]


def run_device(device, shapes, params, tree, cfg):
    opt = P.Shampoo([torch.as_tensor(p, device=device).clone() for p in params], cfg)
    opt.load_state_tree(tree)
    dirs = []
    for g in grads_for(shapes, 1, 2):
        opt.step([torch.as_tensor(x, device=device) for x in g])
        torch.cuda.synchronize()
        dirs.append({(i, b): opt.direction(i, b).cpu().numpy().copy() for (i, b) in opt._pid})
    out = opt.state_tree()
    inv = {(i, b): [e[f"inv_factor{k}"] for k in range(len(e)) if f"inv_factor{k}" in e]
           for i, row in out["params"].items() for b, e in row.items() if e["kind"] == "shampoo"}
    g = opt.guard_stats
    return dirs, inv, (g.primary, g.double_retry, g.fallback_previous, g.fallback_identity)


def well_posed(f, eps, t0) -> bool:
    a = f / (1 - BETA2 ** (t0 + 1))
    noise = 2.2e-16 * np.linalg.norm(a, 2) * np.sqrt(a.shape[0])
    return eps >= 1e3 * noise


ROUTES = {
    "scaled_newton": {},
    "unscaled_newton": {"SHAMPOO_NEWTON_SCALE": "0"},
    "jacobi": {"SHAMPOO_EIG_NEWTON": "0"},
}
_ROUTE_DIRS: dict = {}


@pytest.mark.parametrize("eps", [1e-12, 1e-6])
@pytest.mark.parametrize("route", sorted(ROUTES))
def test_steady_state_routes_vs_oracle(cuda_device, monkeypatch, route, eps):
    shapes = block_shapes()
    for k, v in ROUTES[route].items():
        monkeypatch.setenv(k, v)
    params, tree, cfg, odirs, oinv, oguard = oracle_run("steady", shapes, eps, T0)
    dirs, inv, guard = run_device(cuda_device, shapes, params, tree, cfg)
    worst_dir = max(rel(dirs[s][key], odirs[s][key]) for s in range(2) for key in odirs[s])
    worst_inv = 0.0
    for key, refs in oinv.items():
        st = tree["params"][key[0]][key[1]]
        for k, ref in enumerate(refs):
            if well_posed(st[f"factor{k}"], eps, tree["t"]):
                worst_inv = max(worst_inv, rel(inv[key][k], ref))
    print(f"{route} eps={eps:g}: worst direction {worst_dir:.2e}, worst well-posed inverse {worst_inv:.2e}, "
          f"guard {guard} (oracle {oguard})")
    assert worst_dir <= 1e-3, worst_dir
    assert worst_inv <= 1e-7, worst_inv
    assert guard[0] + guard[1] == oguard[0] + oguard[1] and guard[2:] == oguard[2:]
    # all routes agree with each other (the same matrix function)
    _ROUTE_DIRS.setdefault(eps, {})[route] = dirs
    others = [r for r in _ROUTE_DIRS[eps] if r != route]
    for r in others:
        d = max(rel(dirs[s][key], _ROUTE_DIRS[eps][r][s][key]) for s in range(2) for key in dirs[s])
        assert d <= 1e-3, (route, r, d)


@pytest.mark.parametrize("eps", [1e-12, 1e-6])
def test_early_state_low_rank_route_vs_oracle(cuda_device, eps):
    """Vector factors of structural rank 100 < d (the low-rank range-compression route)."""
    shapes = [s for s in block_shapes() if len(s) == 1 and s[0] >= 128] + [(2048, 512), (512, 1536, 3)]
    params, tree, cfg, odirs, oinv, oguard = oracle_run("early", shapes, eps, 100)
    dirs, inv, guard = run_device(cuda_device, shapes, params, tree, cfg)
    worst_dir = max(rel(dirs[s][key], odirs[s][key]) for s in range(2) for key in odirs[s])
    print(f"low-rank eps={eps:g}: worst direction {worst_dir:.2e}, guard {guard} (oracle {oguard})")
    assert worst_dir <= 1e-3, worst_dir


@pytest.mark.parametrize("eps", [1e-12, 1e-6])
def test_full_resnet50_two_steps_vs_oracle(cuda_device, eps):
    """All 161 ResNet-50 tensors, two steps from t = 0 (refresh at t = 0, stale t = 1), fp32
    gradients, float64 parameters: directions <= 1e-3, parameters <= 1e-6."""
    shapes = [tuple(s) for s in MODEL_SHAPES["resnet50"]]
    rng = np.random.default_rng(0)
    params = [(rng.standard_normal(s) * 0.05).astype(np.float32).astype(np.float64) for s in shapes]
    kw = dict(max_preconditioner_dim=2048, precondition_frequency=F, epsilon=eps)
    oracle = O.OracleShampoo(params, O.OracleConfig(grafting=O.GraftKind.ADAGRAD, **kw))
    opt = P.Shampoo([torch.as_tensor(p, device=cuda_device).clone() for p in params],
                    P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, **kw))
    worst = 0.0
    for g in grads_for(shapes, 1, 2):
        d_ref = oracle.step(g)
        opt.step([torch.as_tensor(x, device=cuda_device) for x in g])
        torch.cuda.synchronize()
        worst = max(worst, max(rel(opt.direction(i, b).cpu().numpy(), ref) for (i, b), ref in d_ref.items()))
    worst_p = max(rel(a.cpu().numpy(), b) for a, b in zip(opt.params(), oracle.params))
    print(f"resnet50 x161 eps={eps:g}: worst direction {worst:.2e}, worst parameter {worst_p:.2e}")
    assert worst <= 1e-3
    # parameters move by lr * p with lr = 0.1 and |p| ~ |W|: their error is ~ the direction error; at
    # eps = 1e-12 the t = 0 factors are rank deficient and the reference's own answer carries the
    # float64 null-space noise (tests/test_gpu_parity.py::test_root_inverse_eigh_matches_reference)
    assert worst_p <= (1e-4 if eps < 1e-9 else 1e-6)
