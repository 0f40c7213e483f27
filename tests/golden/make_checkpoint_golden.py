"""Checkpoint-interop fixtures written by the REAL reference (``minishampoo.checkpoint``).

Run in the build container only (``/root/reference`` does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_checkpoint_golden.py

For each case the reference runs a few steps, writes its JSON-hex checkpoint
(``save_checkpoint``, checkpoint.py:114-126) to ``ref_ckpt_<case>.json``, then
continues from the checkpoint for CONT more steps on recorded gradients;
``ref_ckpt_cont.npz`` holds those gradients and the continued parameters.  The
sharded case writes the union of the group-0 workers' state trees
(train.py:346-353) after ``distributed_step`` on 2 workers, exactly like the
reference trainer, and continues single-process from the merged checkpoint.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from minishampoo.checkpoint import load_checkpoint, save_checkpoint  # noqa: E402
from minishampoo.dist import build_workers, distributed_step  # noqa: E402
from minishampoo.grafting import GraftKind  # noqa: E402
from minishampoo.optim import Shampoo, ShampooConfig  # noqa: E402
from minishampoo.train import _merged_state_tree  # noqa: E402

SHAPES = [(24, 20), (20,), (6, 5, 4), (3, 10), (1, 1)]
CONT = 4
CASES = {
    "double": dict(precision="double"),
    "single": dict(precision="single", epsilon=1e-6),
    "sharded": dict(precision="double"),
}


def config(**kw):
    base = dict(lr=0.05, betas=(0.9, 0.999), momentum=0.9, use_nesterov=True, weight_decay=1e-4,
                grafting=GraftKind.ADAGRAD, precondition_frequency=2, max_preconditioner_dim=16, epsilon=1e-6)
    base.update(kw)
    return ShampooConfig(**base)


def grads(rng, steps):
    return [[(rng.standard_normal(s) * 0.1).astype(np.float32).astype(np.float64) for s in SHAPES]
            for _ in range(steps)]


def main():
    cont = {}
    for case, kw in CASES.items():
        rng = np.random.default_rng(7)
        params = [(rng.standard_normal(s) * 0.5).astype(np.float32).astype(np.float64) for s in SHAPES]
        cfg = config(**kw)
        pre = grads(rng, 5)
        if case == "sharded":
            _, workers = build_workers(params, cfg, world_size=2, group_size=2)
            for g in pre:
                result = distributed_step(workers, g)
            tree = _merged_state_tree(workers)
            cur = [p.copy() for p in result]
            step = workers[0].optimizer.step_count
        else:
            opt = Shampoo([p.copy() for p in params], cfg)
            for g in pre:
                opt.step(g)
            tree = opt.state_tree()
            cur = [p.copy() for p in opt.params()]
            step = opt.step_count
        path = os.path.join(HERE, f"ref_ckpt_{case}.json")
        save_checkpoint(path, step, cur, tree)
        # continue from the file, as a resumed reference run would
        step2, p2, tree2 = load_checkpoint(path)
        opt2 = Shampoo(p2, cfg)
        opt2.load_state_tree(tree2)
        post = grads(rng, CONT)
        for k, g in enumerate(post):
            opt2.step(g)
            for i, x in enumerate(g):
                cont[f"{case}/grad/{k}/{i}"] = x.astype(np.float32)
        for i, p in enumerate(opt2.params()):
            cont[f"{case}/final/{i}"] = p.copy()
        print(case, "step", step, "bytes", os.path.getsize(path))
    np.savez_compressed(os.path.join(HERE, "ref_ckpt_cont.npz"), **cont)


if __name__ == "__main__":
    main()
