"""Generate golden fixtures by running the REAL reference package (``minishampoo``).

Run in the build container only (``/root/reference`` does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Outputs (committed, small):
  plans.npz        block tables + greedy assignments for the benchmark model sets
  trajectories.npz multi-step Shampoo.step runs (params, directions, factors, inverses)
  rootinv.npz      root_inverse_eigh / root_inverse_newton on seeded SPD/PSD matrices

Gradients are drawn as float32 (then up-cast) so the GPU side can consume the
identical values (SURVEY.md §8c "How the harness uses it").
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(HERE, "..", ".."))

from minishampoo import matfun  # noqa: E402
from minishampoo.dist import comm_meter, enumerate_blocks, greedy_assign  # noqa: E402
from minishampoo.grafting import GraftKind  # noqa: E402
from minishampoo.optim import Shampoo, ShampooConfig  # noqa: E402
from minishampoo.precond import LargeDimMethod  # noqa: E402

from paper_2309_06497_b200.model_shapes import MODEL_SHAPES  # noqa: E402

PLAN_CASES = [
    ("resnet50", 2048), ("resnet50", 1024), ("vit_b_16", 1024), ("gpt2_medium", 1024),
    ("mlp", 512), ("mlp", 128),
]
WORLDS = [(1, 1), (2, 2), (4, 4), (8, 8), (8, 4), (8, 2), (4, 2)]


def make_plans(out):
    for model, b in PLAN_CASES:
        shapes = [tuple(s) for s in MODEL_SHAPES[model]]
        blocks = enumerate_blocks(shapes, ShampooConfig(max_preconditioner_dim=b))
        key = f"{model}_b{b}"
        out[f"{key}/param_index"] = np.array([x.param_index for x in blocks], np.int64)
        out[f"{key}/block_index"] = np.array([x.block_index for x in blocks], np.int64)
        out[f"{key}/var_count"] = np.array([x.var_count for x in blocks], np.int64)
        shp = np.zeros((len(blocks), 4), np.int64)
        for j, x in enumerate(blocks):
            shp[j, : len(x.shape)] = x.shape
        out[f"{key}/shape"] = shp
        for world, group in WORLDS:
            plan = greedy_assign([x.var_count for x in blocks], world, group)
            owner = np.zeros(len(blocks), np.int64)
            offset = np.zeros(len(blocks), np.int64)
            for gid, region in plan.buffer_layout.items():
                owner[gid] = region.owner_rank
                offset[gid] = region.byte_offset // 8
            wk = f"{key}/J{world}G{group}"
            out[f"{wk}/owner"] = owner
            out[f"{wk}/offset"] = offset
            out[f"{wk}/counters"] = np.array(plan.counters, np.int64)
            rep = comm_meter(plan, [x.shape for x in blocks], steps=3)  # dist.py:394-423
            out[f"{wk}/comm"] = np.array([rep.bytes_gathered_per_step, rep.world_bytes_per_step,
                                          rep.total_bytes_gathered], np.int64)
            out[f"{wk}/state_scalars"] = np.array(rep.per_worker_state_scalars, np.int64)


TRAJ_SHAPES = [(6, 5), (7,), (3, 4, 5), (2, 3, 3, 1), (1, 1), (9, 4)]

TRAJ_CONFIGS = {
    "adagrad_nesterov": dict(grafting=GraftKind.ADAGRAD, betas=(0.0, 0.999), momentum=0.9,
                             precondition_frequency=3, max_preconditioner_dim=6),
    "adam_beta1_l2": dict(grafting=GraftKind.ADAM, betas=(0.9, 0.99), momentum=0.5,
                          use_nesterov=False, use_decoupled_weight_decay=False,
                          weight_decay=1e-3, precondition_frequency=2, max_preconditioner_dim=5,
                          start_preconditioning_step=1),
    "sgd_sum_nobias": dict(grafting=GraftKind.SGD, betas=(0.0, 1.0), use_bias_correction=False,
                           precondition_frequency=1, max_preconditioner_dim=8, epsilon=1e-6),
    "rmsprop_override": dict(grafting=GraftKind.RMSPROP, exponent_override=2,
                             exponent_multiplier=1.5, precondition_frequency=2,
                             max_preconditioner_dim=4, epsilon=1e-9, lr_schedule="warmup_cosine",
                             warmup_steps=2, total_steps=10),
    "newton_adagrad": dict(grafting=GraftKind.ADAGRAD, solver=matfun.Solver.COUPLED_NEWTON,
                           precondition_frequency=2, max_preconditioner_dim=6, epsilon=1e-6),
    "normalized_adam": dict(grafting=GraftKind.NORMALIZED_ADAM, betas=(0.5, 0.9),
                            precondition_frequency=2, max_preconditioner_dim=6, epsilon=1e-8),
    "normalized_adagrad": dict(grafting=GraftKind.NORMALIZED_ADAGRAD, momentum=0.9,
                               precondition_frequency=3, max_preconditioner_dim=6, epsilon=1e-10),
    "normalized_rmsprop": dict(grafting=GraftKind.NORMALIZED_RMSPROP, grafting_beta2=0.95,
                               betas=(0.0, 0.99), weight_decay=1e-3, use_decoupled_weight_decay=False,
                               precondition_frequency=2, max_preconditioner_dim=5, epsilon=1e-9),
}
TRAJ_STEPS = 6

# large-dimension fallbacks: a dim above max_preconditioner_dim selects ADAGRAD / DIAGONAL
# for that parameter (precond.py:114-158, 282-396); other params stay BLOCKING
FALLBACK_SHAPES = [(9, 4), (13, 3), (2, 11, 3), (6,)]
FALLBACK_CONFIGS = {
    "fallback_adagrad": dict(grafting=GraftKind.ADAGRAD, large_dim_method=LargeDimMethod.ADAGRAD,
                             precondition_frequency=2, max_preconditioner_dim=8, betas=(0.0, 0.99)),
    "fallback_diagonal": dict(grafting=GraftKind.RMSPROP, large_dim_method=LargeDimMethod.DIAGONAL,
                              precondition_frequency=2, max_preconditioner_dim=8, epsilon=1e-6,
                              exponent_multiplier=0.5, betas=(0.5, 0.999)),
    "fallback_diag_sum": dict(grafting=GraftKind.SGD, large_dim_method=LargeDimMethod.DIAGONAL,
                              precondition_frequency=1, max_preconditioner_dim=8, epsilon=1e-8,
                              betas=(0.0, 1.0), start_preconditioning_step=2),
}


def make_trajectories(out, meta):
    cases = [(n, kw, TRAJ_SHAPES) for n, kw in TRAJ_CONFIGS.items()]
    cases += [(n, kw, FALLBACK_SHAPES) for n, kw in FALLBACK_CONFIGS.items()]
    for name, kw, shapes in cases:
        cfg = ShampooConfig(lr=0.05, **kw)
        rng = np.random.default_rng(0)
        params = [(rng.standard_normal(s) * 0.5).astype(np.float32) for s in shapes]
        grng = np.random.default_rng(1)
        grads = [[(grng.standard_normal(s) * 0.1).astype(np.float32) for s in shapes]
                 for _ in range(TRAJ_STEPS)]
        opt = Shampoo([p.astype(np.float64) for p in params], cfg)
        captured = {}
        orig = opt.apply_directions

        def capture(directions, t, _orig=orig):
            captured.clear()
            captured.update({k: np.array(v) for k, v in directions.items()})
            return _orig(directions, t)

        opt.apply_directions = capture
        for i, p in enumerate(params):
            out[f"{name}/init/{i}"] = p
        for t in range(TRAJ_STEPS):
            for i, g in enumerate(grads[t]):
                out[f"{name}/grad/{t}/{i}"] = g
            opt.step([g.astype(np.float64) for g in grads[t]])
            for (i, b), d in captured.items():
                out[f"{name}/dir/{t}/{i}/{b}"] = d
            for i, p in enumerate(opt.params()):
                out[f"{name}/param/{t}/{i}"] = p.copy()
        tree = opt.state_tree()
        for i, pt in tree["params"].items():
            for b, entry in pt.items():
                for k, v in entry.items():
                    if isinstance(v, np.ndarray):
                        out[f"{name}/state/{i}/{b}/{k}"] = v
        meta[name] = {"config": {k: (v.value if hasattr(v, "value") else v) for k, v in kw.items()},
                      "guard": vars(opt.guard_stats), "shapes": [list(x) for x in shapes]}


def make_rootinv(out):
    rng = np.random.default_rng(5)
    cases = []
    for n in (1, 3, 8, 33, 64, 100):
        q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = np.exp(np.linspace(0.0, np.log(1e6), n)) / 1e6
        a = (q * lam) @ q.T
        cases.append((f"spd{n}", (a + a.T) / 2))
    for n, r in ((16, 1), (40, 5), (70, 3)):
        g = rng.standard_normal((n, r))
        a = g @ g.T
        cases.append((f"psd{n}r{r}", (a + a.T) / 2))
    for name, a in cases:
        out[f"{name}/a"] = a
        for p in (2, 4, 6):
            for eps in (1e-12, 1e-6):
                req = matfun.RootInverseRequest(a, root_p=p, epsilon=eps)
                out[f"{name}/eigh/p{p}/e{eps:g}"] = matfun.root_inverse_eigh(req)
        if name.startswith("spd") and a.shape[0] <= 64:
            for p in (2, 4):
                req = matfun.RootInverseRequest(a, root_p=p, epsilon=1e-6,
                                                solver=matfun.Solver.COUPLED_NEWTON)
                x, tr = matfun.root_inverse_newton(req)
                out[f"{name}/newton/p{p}"] = x
                out[f"{name}/newton/p{p}/iters"] = np.array(tr.iterations)


def main():
    plans, traj, rinv, meta = {}, {}, {}, {}
    make_plans(plans)
    np.savez_compressed(os.path.join(HERE, "plans.npz"), **plans)
    if "--plans-only" in sys.argv:
        return
    make_trajectories(traj, meta)
    make_rootinv(rinv)
    np.savez_compressed(os.path.join(HERE, "trajectories.npz"), **traj)
    np.savez_compressed(os.path.join(HERE, "rootinv.npz"), **rinv)
    with open(os.path.join(HERE, "trajectories.json"), "w") as fh:
        json.dump({"steps": TRAJ_STEPS, "shapes": TRAJ_SHAPES, "configs": meta}, fh, indent=1)
    print("wrote", len(plans), len(traj), len(rinv), "arrays")


if __name__ == "__main__":
    main()
