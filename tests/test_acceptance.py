"""Reference acceptance #11 (test_acceptance.py:288-327): preconditioning beats tuned SGD.

The reference trainer's MLP task (tests/mlp_task.py, pinned below to the real reference) trained
on the GPU with torch autograd (float64) and this package's DistributedShampoo: 2000 steps, batch 64,
block cap 32, four refresh intervals and four SGD learning rates (start_preconditioning_step = inf).
Checked against the reference's own final losses (tests/golden/acceptance11.json) and the test's
acceptance bounds: Shampoo at f = 50 <= the best SGD, refresh-interval spread < 5%, < 120 s.
"""

from __future__ import annotations

import json
import math
import os
import time

import numpy as np
import pytest

from tests.conftest import ROOT
from tests.mlp_task import acceptance11_task, batch_indices, init_weights

GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "acceptance11.json")))


def test_mlp_task_pinned():
    """tests/mlp_task.py reproduces the reference's data, split, initialisation and batches."""
    x, y, w0 = acceptance11_task(0)
    pin = GOLD["pin"]
    assert len(x) == pin["n_train"]
    assert x.sum() == pytest.approx(pin["train_x_sum"], rel=1e-12, abs=1e-9)
    assert (x ** 2).sum() == pytest.approx(pin["train_x_sq"], rel=1e-12)
    assert x[0, 0] == pin["train_x_00"]
    assert int(y.sum()) == pin["train_y_sum"]
    for w, s, q in zip(w0, pin["w0_sum"], pin["w0_sq"]):
        assert w.sum() == pytest.approx(s, rel=1e-12, abs=1e-12) and (w ** 2).sum() == pytest.approx(q, rel=1e-12)
    assert x[batch_indices(0, 0, len(x), 64)].sum() == pytest.approx(pin["batch0_x_sum"], rel=1e-12, abs=1e-9)
    assert int(y[batch_indices(0, 1999, len(x), 64)].sum()) == pin["batch1999_y_sum"]


def _train(torch, P, x, y, idx, cfg_kw, dev):
    w = [torch.tensor(a, dtype=torch.float64, device=dev, requires_grad=True) for a in init_weights([32, 64, 10], 0)]
    kw = dict(cfg_kw)
    opt = P.DistributedShampoo(w, check_finite="deferred", **kw)
    losses = torch.empty(idx.shape[0], dtype=torch.float64, device=dev)
    for t in range(idx.shape[0]):
        b = idx[t]
        logits = torch.relu(x[b] @ w[0].T) @ w[1].T
        loss = torch.nn.functional.cross_entropy(logits, y[b])
        opt.zero_grad(set_to_none=False)
        loss.backward()
        opt.step()
        losses[t] = loss.detach()
    opt.engine.synchronize()
    return losses.cpu().numpy()


@pytest.mark.gpu
def test_11_preconditioning_beats_tuned_sgd(cuda_device):
    import torch

    import paper_2309_06497_b200 as P

    started = time.perf_counter()
    xs, ys, _ = acceptance11_task(0)
    x = torch.tensor(xs, dtype=torch.float64, device=cuda_device)
    y = torch.tensor(ys, dtype=torch.int64, device=cuda_device)
    idx = torch.tensor(np.stack([batch_indices(0, t, len(xs), 64) for t in range(2000)]), device=cuda_device)
    c = GOLD["config"]
    base = dict(lr=c["lr"], betas=tuple(c["betas"]), epsilon=c["epsilon"], momentum=c["momentum"],
                use_nesterov=c["use_nesterov"], weight_decay=c["weight_decay"],
                use_decoupled_weight_decay=c["use_decoupled_weight_decay"],
                use_bias_correction=c["use_bias_correction"], max_preconditioner_dim=c["max_preconditioner_dim"],
                precondition_frequency=c["precondition_frequency"],
                start_preconditioning_step=c["start_preconditioning_step"],
                exponent_override=c["exponent_override"], exponent_multiplier=c["exponent_multiplier"],
                grafting=c["grafting"], grafting_epsilon=c["grafting_epsilon"], grafting_beta2=c["grafting_beta2"],
                solver=c["solver"], newton_tolerance=c["newton_tolerance"], large_dim_method=c["large_dim_method"],
                precision=c["precision"])
    assert base["max_preconditioner_dim"] == 32
    runs = {}
    traj50 = None
    for freq in (1, 20, 50, 100):
        losses = _train(torch, P, x, y, idx, {**base, "precondition_frequency": freq}, cuda_device)
        runs[f"shampoo_f{freq}"] = float(losses[-100:].mean())
        if freq == 50:
            traj50 = losses
    for lr in (0.3, 0.1, 0.03, 0.01):
        losses = _train(torch, P, x, y, idx, {**base, "lr": lr, "start_preconditioning_step": math.inf}, cuda_device)
        runs[f"sgd_lr{lr}"] = float(losses[-100:].mean())
    elapsed = time.perf_counter() - started
    # same training as the reference: per-step losses of the f = 50 run track the reference's, and
    # every final (tail-mean) loss agrees
    ref50 = np.asarray(GOLD["loss_f50"])
    dev50 = np.abs(traj50 - ref50)
    print("f50 per-step |loss - reference| max over steps <100/<200/<500/<1000/all:",
          [float(dev50[:k].max()) for k in (100, 200, 500, 1000, 2000)])
    print("final losses (ours, reference):", {k: (round(v, 5), round(GOLD["runs"][k], 5)) for k, v in runs.items()})
    # step-by-step parity while the runs are still close (measured 2.9e-7 over the first 500 steps)
    assert dev50[:500].max() <= 1e-5
    # after that the training is chaotic: the REFERENCE itself moves its f = 50 tail loss by 0.23% (and
    # its step-999 loss by 2.5%) when W0 is scaled by 1 + 1e-9; SGD runs (no root inverse) and the
    # f = 1 run agree to 5 digits, the others within a few 1e-3 -- bound 1.5%
    for k, v in runs.items():
        tol = 1e-6 if k.startswith("sgd") else 1.5e-2
        assert abs(v - GOLD["runs"][k]) <= tol * GOLD["runs"][k], (k, v, GOLD["runs"][k])
    # the acceptance bounds (test_acceptance.py:318-321)
    best_sgd = min(v for k, v in runs.items() if k.startswith("sgd"))
    by_freq = [v for k, v in runs.items() if k.startswith("shampoo")]
    spread = (max(by_freq) - min(by_freq)) / min(by_freq)
    assert runs["shampoo_f50"] <= best_sgd, runs
    assert spread < 0.05, runs
    assert elapsed < 120.0, elapsed
