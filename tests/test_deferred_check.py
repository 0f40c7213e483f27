"""Deferred non-finite check (check_finite="deferred"): no host synchronisation per step.

The check predicates every state-writing kernel of the step on a device word; a skipped step
raises NonFiniteGradientError at the NEXT call (optim.py:362-366 semantics, one call late) with
the step counter rolled back, and the device state equals the state before the bad step.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2309_06497_b200 as P

pytestmark = pytest.mark.gpu

SHAPES = [(24, 20), (40,), (6, 5, 4), (300, 9), (130, 70)]


def _setup(dev, mode, graft=P.GraftKind.ADAM, f=3, **kw):
    rng = np.random.default_rng(5)
    params = [torch.as_tensor(rng.standard_normal(s).astype(np.float32), device=dev) for s in SHAPES]
    cfg = P.ShampooConfig(lr=0.05, betas=(0.9, 0.999), momentum=0.9, weight_decay=1e-4, grafting=graft,
                          precondition_frequency=f, max_preconditioner_dim=64, epsilon=1e-10, **kw)
    return P.Shampoo(params, cfg, check_finite=mode)


def _grads(dev, n, seed=9):
    rng = np.random.default_rng(seed)
    return [[torch.as_tensor((0.1 * rng.standard_normal(s)).astype(np.float32), device=dev) for s in SHAPES]
            for _ in range(n)]


def _tree_equal(a, b):
    assert a["t"] == b["t"]
    assert a["params"].keys() == b["params"].keys()
    for i, pa in a["params"].items():
        pb = b["params"][i]
        assert pa.keys() == pb.keys()
        for blk, ba in pa.items():
            bb = pb[blk]
            for k, v in ba.items():
                if isinstance(v, np.ndarray):
                    assert np.array_equal(v, bb[k]), k
                else:
                    assert v == bb[k], k


@pytest.mark.parametrize("graft", [P.GraftKind.ADAM, P.GraftKind.ADAGRAD, P.GraftKind.NORMALIZED_ADAGRAD])
def test_deferred_trajectory_bitwise_equals_strict(cuda_device, graft):
    gs = _grads(cuda_device, 8)
    strict, lazy = _setup(cuda_device, True, graft), _setup(cuda_device, "deferred", graft)
    for g in gs:
        strict.step(g)
        lazy.step(g)
    lazy.synchronize()
    for a, b in zip(strict.params(), lazy.params()):
        assert torch.equal(a, b)
    _tree_equal(strict.state_tree(), lazy.state_tree())


@pytest.mark.parametrize("bad_at", [1, 4])  # plain steps (refreshes at t = 0, 3, 6)
def test_deferred_nonfinite_skips_step_and_raises_next_call(cuda_device, bad_at):
    gs = _grads(cuda_device, 7)
    ref = _setup(cuda_device, True)
    for g in gs[:bad_at] + gs[bad_at + 1:]:  # the run that never saw the bad gradients
        ref.step(g)
    opt = _setup(cuda_device, "deferred")
    for g in gs[:bad_at]:
        opt.step(g)
    opt.synchronize()
    before = opt.state_tree()
    p_before = [p.clone() for p in opt.params()]
    bad = [g.clone() for g in gs[bad_at]]
    bad[2][1, 2, 3] = float("inf")
    opt.step(bad)  # returns: the check result is read one call late
    with pytest.raises(P.NonFiniteGradientError):
        opt.step(gs[bad_at + 1])  # raised before this step is launched
    assert opt.step_count == bad_at
    for a, b in zip(opt.params(), p_before):
        assert torch.equal(a, b)
    _tree_equal(before, opt.state_tree())
    for g in gs[bad_at + 1:]:
        opt.step(g)
    opt.synchronize()
    for a, b in zip(opt.params(), ref.params()):
        assert torch.equal(a, b)
    _tree_equal(ref.state_tree(), opt.state_tree())


def test_deferred_refresh_step_checked_eagerly(cuda_device):
    gs = _grads(cuda_device, 4)
    opt = _setup(cuda_device, "deferred")
    for g in gs[:3]:
        opt.step(g)
    bad = [g.clone() for g in gs[3]]
    bad[0][0, 0] = float("nan")
    with pytest.raises(P.NonFiniteGradientError):
        opt.step(bad)  # t = 3 is a refresh step: raised by the step itself
    assert opt.step_count == 3


def test_deferred_check_via_facade(cuda_device):
    torch.manual_seed(0)
    model = torch.nn.Linear(30, 12).to(cuda_device)
    opt = P.DistributedShampoo(model.parameters(), lr=0.05, max_preconditioner_dim=32,
                               precondition_frequency=2, check_finite="deferred")
    x = torch.randn(16, 30, device=cuda_device)
    for _ in range(3):
        opt.zero_grad()
        model(x).square().mean().backward()
        opt.step()
    w = model.weight.detach().clone()
    opt.zero_grad()
    model(x).square().mean().backward()
    model.weight.grad[0, 0] = float("nan")
    opt.step()  # t = 3: plain step, deferred
    with pytest.raises(P.NonFiniteGradientError):
        opt.step()
    assert torch.equal(model.weight.detach(), w)
    assert opt.step_count == 3
