"""World-2 runs of the device step through ``DistributedShampoo`` (the NCCL path never ran).

Two processes, each with a device optimizer context that owns half of the blocks (greedy plan,
dist.py:133-183), directions exchanged by the product's ``GroupExchange``:

* ``nccl``: one GPU per rank -- skipped when fewer than 2 GPUs are visible (the gpurun pool gives 1);
* ``gloo``: both ranks on cuda:0, host-staged collectives -- runs on the one-GPU box and exercises the
  same sharded device path (owned-only state, region fill, all-gather, apply-all).

Checks (test_dist.py:173-221 pattern): J = 2 parameters equal the single-process (J = 1) run to
1e-12, replicas are bit-identical, the replica drift check passes and then raises
``DivergedReplicasError`` once a replica is perturbed, and the reduce-scatter gradient path
(``reduce_gradients="mean"``) from per-rank local gradients equals the single-process step on the
mean gradient.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

SHAPES = [(24, 16), (16,), (6, 5, 4), (1, 1), (40, 9), (33,)]
KW = dict(lr=0.05, max_preconditioner_dim=16, precondition_frequency=2, epsilon=1e-10, grafting="adagrad")
STEPS = 5


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs():
    rng = np.random.default_rng(0)
    params = [rng.standard_normal(s) * 0.5 for s in SHAPES]
    grads = [[[rng.standard_normal(s) * 0.1 for s in SHAPES] for _ in range(2)] for _ in range(STEPS)]
    return params, grads  # grads[t][r]: rank r's local gradient at step t


def _single_process(device, mode):
    import paper_2309_06497_b200 as P

    params, grads = _inputs()
    ps = [torch.nn.Parameter(torch.as_tensor(p, device=device)) for p in params]
    opt = P.DistributedShampoo(ps, **KW)
    for t in range(STEPS):
        for p, g0, g1 in zip(ps, grads[t][0], grads[t][1]):
            g = g0 if mode == "global" else (g0 + g1) / 2
            p.grad = torch.as_tensor(g, device=device)
        opt.step()
    torch.cuda.synchronize()
    return [p.detach().cpu().numpy() for p in ps]


def _worker(rank, world, port, backend, mode, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dev = torch.device("cuda", rank if backend == "nccl" else 0)
    torch.cuda.set_device(dev)
    if backend == "nccl":
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2309_06497_b200 as P

        params, grads = _inputs()
        ps = [torch.nn.Parameter(torch.as_tensor(p, device=dev)) for p in params]
        opt = P.DistributedShampoo(ps, reduce_gradients=None if mode == "global" else "mean",
                                   check_replicas_every=1, **KW)
        owned = sorted(opt.engine.owned_ids)
        for t in range(STEPS):
            for p, g0, g1 in zip(ps, grads[t][0], grads[t][1]):
                g = g0 if mode == "global" else (g0, g1)[rank]  # "local": each rank its own gradient
                p.grad = torch.as_tensor(g, device=dev)
            opt.step()
        torch.cuda.synchronize()
        result = [p.detach().cpu().numpy() for p in ps]
        diverged = None
        if mode == "global":
            if rank == 1:
                with torch.no_grad():
                    ps[0][0, 0] += 1e-6
            try:
                opt.exchange.check_replicas(ps)
                diverged = False
            except P.DivergedReplicasError:
                diverged = True
        out[rank] = (result, owned, diverged, opt.exchange.bytes_per_step)
    finally:
        dist.destroy_process_group()


def _run(backend, mode):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, backend, mode, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    return out[0], out[1]


BACKENDS = [
    "gloo",
    pytest.param("nccl", marks=pytest.mark.skipif(
        not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")),
]


@pytest.mark.parametrize("backend", BACKENDS)
def test_world2_matches_single_process_and_replicas_identical(cuda_device, backend):
    (r0, own0, div0, nbytes), (r1, own1, div1, _) = _run(backend, "global")
    ref = _single_process(cuda_device, "global")
    assert own0 and own1 and not set(own0) & set(own1)  # disjoint owned blocks, both non-empty
    for a, b, c in zip(r0, r1, ref):
        assert np.array_equal(a, b)  # replicas bit-identical (test_dist.py:187-196)
        assert np.abs(a - c).max() <= 1e-12  # world-size invariance (test_dist.py:173-185)
    assert nbytes > 0
    assert div0 is True and div1 is True  # the perturbed replica is detected on every rank


@pytest.mark.parametrize("backend", BACKENDS)
def test_world2_reduced_local_gradients_match_mean_gradient(cuda_device, backend):
    (r0, _, _, _), (r1, _, _, _) = _run(backend, "local")
    ref = _single_process(cuda_device, "mean")
    for a, b, c in zip(r0, r1, ref):
        assert np.array_equal(a, b)
        assert np.abs(a - c).max() <= 1e-12
