"""Golden values for acceptance #11 (test_acceptance.py:288-327) from the REAL reference.

Build container only:  PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_acceptance11.py

Records (tests/golden/acceptance11.json): checksums of the reference's data / init / batches (pin
tests/mlp_task.py), the ShampooConfig the acceptance test trains with, and the reference's final
tail-mean loss for every run of the test (4 refresh intervals, 4 SGD learning rates) plus the
per-step loss of the frequency-50 run.
"""

from __future__ import annotations

import json
import math
import os
import sys
import time
from dataclasses import asdict, replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from minishampoo.config import RunConfig  # noqa: E402
from minishampoo.train import Mlp, batch_at, make_synthetic_classes, prepare_bundle, run_training  # noqa: E402


def main():
    features, labels = make_synthetic_classes(seed=0, classes=10, dim=32, count=8192)
    bundle = prepare_bundle(features, labels, seed=0)
    base = RunConfig(max_preconditioner_dim=32).to_shampoo_config()
    w0 = Mlp.initialize([32, 64, 10], "relu", seed=0).weights
    b0 = batch_at(bundle, 0, 0, 64)
    b1999 = batch_at(bundle, 0, 1999, 64)
    out = {
        "pin": {
            "train_x_sum": float(bundle.train_x.sum()), "train_x_sq": float((bundle.train_x ** 2).sum()),
            "train_x_00": float(bundle.train_x[0, 0]), "train_y_sum": int(bundle.train_y.sum()),
            "n_train": int(len(bundle.train_x)),
            "w0_sum": [float(w.sum()) for w in w0], "w0_sq": [float((w ** 2).sum()) for w in w0],
            "batch0_x_sum": float(b0[0].sum()), "batch1999_y_sum": int(b1999[1].sum()),
        },
        "config": {k: (v.value if hasattr(v, "value") else (None if isinstance(v, float) and math.isinf(v) else v))
                   for k, v in asdict(base).items()},
        "runs": {},
    }

    def final_loss(config, keep=False):
        model = Mlp.initialize([32, 64, 10], "relu", seed=0)
        result = run_training(bundle, model, config, steps=2000, batch_size=64, seed=0)
        losses = [row.loss for row in result.metrics]
        tail = losses[-100:]
        return sum(tail) / len(tail), (losses if keep else None)

    t0 = time.perf_counter()
    for freq in (1, 20, 50, 100):
        v, traj = final_loss(replace(base, precondition_frequency=freq), keep=freq == 50)
        out["runs"][f"shampoo_f{freq}"] = v
        if traj:
            out["loss_f50"] = traj
    for lr in (0.3, 0.1, 0.03, 0.01):
        v, _ = final_loss(replace(base, lr=lr, start_preconditioning_step=math.inf))
        out["runs"][f"sgd_lr{lr}"] = v
    out["reference_seconds"] = time.perf_counter() - t0
    with open(os.path.join(HERE, "acceptance11.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(json.dumps(out["runs"], indent=1), out["reference_seconds"])


if __name__ == "__main__":
    main()
