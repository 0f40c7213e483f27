"""The torch.optim facade ``DistributedShampoo`` (north_star's named API).

Single process: ``step()`` from ``p.grad`` equals the engine step bit for bit, closures return their
loss, ``state_dict`` / ``load_state_dict`` resume bitwise, torch LR schedulers drive the applied lr,
and a short trajectory matches the float64 oracle.  Multi-process (world 2): see
tests/test_distributed_device.py.
"""

from __future__ import annotations

import copy

import numpy as np
import pytest
import torch

import paper_2309_06497_b200 as P
from oracle import shampoo_oracle as O

pytestmark = pytest.mark.gpu

SHAPES = [(16, 12), (12,), (4, 3, 5), (1, 1), (40, 9)]
KW = dict(lr=0.05, max_preconditioner_dim=16, precondition_frequency=2, epsilon=1e-10, weight_decay=1e-3)


def make_params(device, seed=0):
    rng = np.random.default_rng(seed)
    return [torch.nn.Parameter(torch.as_tensor(rng.standard_normal(s) * 0.5, device=device)) for s in SHAPES]


def grad_seq(steps, seed=1):
    rng = np.random.default_rng(seed)
    return [[rng.standard_normal(s) * 0.1 for s in SHAPES] for _ in range(steps)]


def set_grads(params, grads, device):
    for p, g in zip(params, grads):
        p.grad = torch.as_tensor(g, device=device)


def test_facade_step_equals_engine_step(cuda_device):
    pa, pb = make_params(cuda_device), make_params(cuda_device)
    opt = P.DistributedShampoo(pa, grafting="adagrad", **KW)
    eng = P.Shampoo([p.data for p in pb], P.ShampooConfig(grafting=P.GraftKind.ADAGRAD, **KW))
    for g in grad_seq(5):
        set_grads(pa, g, cuda_device)
        opt.step()
        eng.step([torch.as_tensor(x, device=cuda_device) for x in g])
    torch.cuda.synchronize()
    for a, b in zip(pa, pb):
        assert torch.equal(a.data, b.data)
    assert opt.step_count == 5


def test_facade_matches_oracle_trajectory(cuda_device):
    params = make_params(cuda_device)
    init = [p.detach().cpu().numpy().copy() for p in params]
    opt = P.DistributedShampoo(params, grafting="adam", betas=(0.9, 0.999), **KW)
    ref = O.OracleShampoo(init, O.OracleConfig(grafting=O.GraftKind.ADAM, betas=(0.9, 0.999), **KW))
    for g in grad_seq(6):
        set_grads(params, g, cuda_device)
        opt.step()
        ref.step(g)
    torch.cuda.synchronize()
    for a, b in zip(params, ref.params):  # parameters <= 1e-6 relative, as the reference trajectories
        a = a.detach().cpu().numpy()
        assert np.linalg.norm(a - b) <= 1e-6 * np.linalg.norm(b)


def test_facade_closure_returns_loss(cuda_device):
    params = make_params(cuda_device)
    opt = P.DistributedShampoo(params, **KW)
    target = [torch.zeros_like(p) for p in params]

    def closure():
        opt.zero_grad()
        loss = sum(((p - t) ** 2).sum() for p, t in zip(params, target))
        loss.backward()
        return loss

    l0 = float(opt.step(closure))
    for _ in range(5):
        l1 = float(opt.step(closure))
    assert np.isfinite(l0) and l1 < l0  # a quadratic bowl: the loss goes down


def test_facade_state_dict_resume_bitwise(cuda_device):
    pa = make_params(cuda_device)
    opt = P.DistributedShampoo(pa, grafting="rmsprop", **KW)
    seq = grad_seq(7)
    for g in seq[:3]:
        set_grads(pa, g, cuda_device)
        opt.step()
    sd = copy.deepcopy(opt.state_dict())
    saved = [p.detach().clone() for p in pa]
    for g in seq[3:]:
        set_grads(pa, g, cuda_device)
        opt.step()
    pb = [torch.nn.Parameter(s.clone()) for s in saved]
    opt2 = P.DistributedShampoo(pb, grafting="rmsprop", **KW)
    opt2.load_state_dict(sd)
    assert opt2.step_count == 3
    for g in seq[3:]:
        set_grads(pb, g, cuda_device)
        opt2.step()
    torch.cuda.synchronize()
    for a, b in zip(pa, pb):
        assert torch.equal(a.data, b.data)


def test_facade_lr_scheduler_drives_update(cuda_device):
    """torch LR schedulers write param_groups[0]['lr']; the facade applies it (W -= lr * p)."""
    pa, pb = make_params(cuda_device), make_params(cuda_device)
    opt = P.DistributedShampoo(pa, **KW)
    sched = torch.optim.lr_scheduler.LambdaLR(opt, lambda t: 0.5 ** t)
    eng = P.Shampoo([p.data for p in pb], P.ShampooConfig(**KW))
    for t, g in enumerate(grad_seq(4)):
        assert opt.current_lr() == pytest.approx(KW["lr"] * 0.5 ** t)
        set_grads(pa, g, cuda_device)
        opt.step()
        sched.step()
        eng.step([torch.as_tensor(x, device=cuda_device) for x in g], lr=KW["lr"] * 0.5 ** t)
    torch.cuda.synchronize()
    for a, b in zip(pa, pb):
        assert torch.equal(a.data, b.data)
    # lr = 0 leaves the parameters untouched (the state still advances)
    for group in opt.param_groups:
        group["lr"] = 0.0
    before = [p.detach().clone() for p in pa]
    set_grads(pa, grad_seq(1, seed=9)[0], cuda_device)
    opt.step()
    for a, b in zip(pa, before):
        assert torch.equal(a.data, b)


def test_facade_warmup_cosine_schedule(cuda_device):
    """lr_schedule="warmup_cosine": lr_at(t) (optim.py:133-151) scaled by group lr / base lr."""
    params = make_params(cuda_device)
    kw = dict(KW, lr_schedule="warmup_cosine", warmup_steps=2, total_steps=6)
    opt = P.DistributedShampoo(params, **kw)
    cfg = P.ShampooConfig(**kw)
    for t, g in enumerate(grad_seq(3)):
        assert opt.current_lr() == pytest.approx(P.lr_at(cfg, t))
        set_grads(params, g, cuda_device)
        opt.step()
    opt.param_groups[0]["lr"] = KW["lr"] / 2
    assert opt.current_lr() == pytest.approx(P.lr_at(cfg, 3) / 2)


def test_facade_missing_grad_is_zero_gradient(cuda_device):
    pa, pb = make_params(cuda_device), make_params(cuda_device)
    opt = P.DistributedShampoo(pa, **KW)
    eng = P.Shampoo([p.data for p in pb], P.ShampooConfig(**KW))
    g = grad_seq(1)[0]
    set_grads(pa, g, cuda_device)
    pa[1].grad = None
    opt.step()
    g[1] = np.zeros_like(g[1])
    eng.step([torch.as_tensor(x, device=cuda_device) for x in g])
    for a, b in zip(pa, pb):
        assert torch.equal(a.data, b.data)


def test_facade_rejects_bad_arguments(cuda_device):
    params = make_params(cuda_device)
    with pytest.raises(ValueError):
        P.DistributedShampoo(params, betas=(1.0, 0.999))
    with pytest.raises(ValueError):
        P.DistributedShampoo(params, reduce_gradients="max")
    with pytest.raises(ValueError):
        P.DistributedShampoo(params, num_trainers_per_group=2)  # needs torch.distributed
    opt = P.DistributedShampoo(params, **KW)
    set_grads(params, grad_seq(1)[0], cuda_device)
    params[0].grad[0, 0] = float("nan")
    before = [p.detach().clone() for p in params]
    with pytest.raises(P.NonFiniteGradientError):
        opt.step()
    for a, b in zip(params, before):
        assert torch.equal(a.data, b)
    assert opt.step_count == 0
