"""Multi-process (gloo, CPU) tests of the sharded-step host logic (dist.py:133-369).

Each rank builds the plan with the C++ planner (no communication), fills ITS region of the padded
gather buffer with the directions of the blocks it owns (directions from the CPU oracle -- test
infrastructure), and runs the product's ``GroupExchange`` all-gather.  The gathered buffer must
equal, bit for bit, the buffer a single process builds for all blocks; replicas across groups must
agree.  World sizes 2 and 4 (J_G = 2 and 4).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import shampoo_oracle as O

SHAPES = [(6, 4), (5,), (3, 3), (7, 2, 3), (1, 1)]
MAX_DIM = 4


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _reference_buffer(plan_scalars, offsets, blocks, steps):
    """Single-process oracle: directions of ALL blocks for `steps` steps, laid out by the plan."""
    rng = np.random.default_rng(0)
    params = [rng.standard_normal(s) for s in SHAPES]
    cfg = O.OracleConfig(lr=0.05, betas=(0.9, 0.999), grafting=O.GraftKind.ADAGRAD, precondition_frequency=1,
                         max_preconditioner_dim=MAX_DIM)
    opt = O.OracleShampoo(params, cfg)
    grng = np.random.default_rng(1)
    bufs = []
    for _ in range(steps):
        grads = [grng.standard_normal(s) for s in SHAPES]
        dirs = opt.step(grads)
        buf = np.zeros(plan_scalars)
        for b in blocks:
            d = dirs[(b.param_index, b.block_index)].reshape(-1)
            buf[offsets[b.block_id]: offsets[b.block_id] + d.size] = d
        bufs.append(buf)
    return bufs


def _worker(rank, world, group, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2309_06497_b200 as P
        from paper_2309_06497_b200.distributed import GroupExchange

        plan = P.NativePlan(SHAPES, MAX_DIM, P.LargeDimMethod.BLOCKING, world, group)
        ex = GroupExchange(group)
        assert ex.group_size == group
        mp_ = plan.max_payload
        blocks = O.enumerate_blocks(SHAPES, MAX_DIM)
        offsets = [b.gather_offset for b in plan.blocks_info]
        ref = _reference_buffer(group * mp_, offsets, blocks, steps=3)
        owned = plan.owned_ids(rank)
        # the rank's oracle worker: state only for owned blocks (optim.py:205-210)
        rng = np.random.default_rng(0)
        params = [rng.standard_normal(s) for s in SHAPES]
        cfg = O.OracleConfig(lr=0.05, betas=(0.9, 0.999), grafting=O.GraftKind.ADAGRAD,
                             precondition_frequency=1, max_preconditioner_dim=MAX_DIM)
        pairs = {(blocks[i].param_index, blocks[i].block_index) for i in owned}
        opt = O.OracleShampoo(params, cfg, owned=pairs)
        grng = np.random.default_rng(1)
        ok = True
        for t in range(3):
            grads = [grng.standard_normal(s) for s in SHAPES]
            dirs = opt.step(grads)  # computes owned blocks only (and applies them locally)
            buf = torch.zeros(group * mp_, dtype=torch.float64)
            for i in owned:
                d = torch.as_tensor(dirs[(blocks[i].param_index, blocks[i].block_index)].reshape(-1))
                buf[offsets[i]: offsets[i] + d.numel()] = d
            # padding of my region stays zero (dist.py:192)
            ex(buf, rank % group, mp_)
            ok &= bool(np.array_equal(buf.numpy(), ref[t]))
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,group", [(2, 2), (4, 2), (4, 4)])
def test_group_allgather_matches_single_process(world, group):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, group, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert dict(out) == {r: 1 for r in range(world)}


def _reduce_worker(rank, world, group, port, out):
    """GroupExchange.reduce_gradients: after packing LOCAL gradients in the gather
    layout and reducing, this rank's region holds the sum over ALL ranks of the gradients of the blocks
    it owns (reduce-scatter in the group + all-reduce across replica groups); the non-finite flag is a
    max over ranks."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2309_06497_b200 as P
        from paper_2309_06497_b200.distributed import GroupExchange

        plan = P.NativePlan(SHAPES, MAX_DIM, P.LargeDimMethod.BLOCKING, world, group)
        ex = GroupExchange(group)
        mp_ = plan.max_payload
        info = plan.blocks_info

        def packed(r):  # rank r's local gradients in the gather layout (the device pack, restated)
            g = np.random.default_rng(100 + r)
            buf = np.zeros(group * mp_)
            for b in info:
                buf[b.gather_offset: b.gather_offset + b.var_count] = g.standard_normal(b.var_count)
            return buf

        buf = torch.as_tensor(packed(rank))
        ex.reduce_gradients(buf, rank % group, mp_)
        total = sum(packed(r) for r in range(world))
        gr = rank % group
        mine = slice(gr * mp_, (gr + 1) * mp_)
        ok = bool(np.allclose(buf.numpy()[mine], total[mine], rtol=1e-13, atol=1e-13))
        flag = torch.tensor([1 if rank == world - 1 else 0], dtype=torch.int32)
        ex.max_flag(flag)
        ok &= int(flag.item()) == 1
        out[rank] = int(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,group", [(2, 2), (4, 2), (4, 4)])
def test_gradient_reduce_to_owners(world, group):
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_reduce_worker, args=(r, world, group, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    assert dict(out) == {r: 1 for r in range(world)}
