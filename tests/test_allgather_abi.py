"""shampoo_allgather: the C-ABI exchange step (dist.py:350-359) over an NCCL communicator.

One GPU in this pool: a single-rank communicator (ncclCommInitRank with nranks = 1, through ctypes
on the NCCL the process already has loaded) drives the same in-place all-gather call a multi-rank
C user makes; a step composed of the C-ABI phases + shampoo_allgather must equal Shampoo.step
bitwise.  The 2-rank exchange is covered by the gloo tests of GroupExchange and, with >= 2 GPUs,
tests/test_distributed_device.py.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2309_06497_b200 as P
from paper_2309_06497_b200 import _native as N

pytestmark = pytest.mark.gpu


class _UniqueId(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


def _nccl_comm_1rank():
    torch.cuda.init()
    nccl = C.CDLL("libnccl.so.2")  # the copy torch loaded (or the system one)
    uid = _UniqueId()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    return nccl, comm


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_allgather_abi_step_equals_step(cuda_device, dtype):
    nccl, comm = _nccl_comm_1rank()
    try:
        rng = np.random.default_rng(2)
        shapes = [(20, 12), (9,), (3, 4, 5)]
        params = [rng.standard_normal(s) for s in shapes]
        grads = [[rng.standard_normal(s) * 0.1 for s in shapes] for _ in range(4)]
        cfg = P.ShampooConfig(lr=0.05, max_preconditioner_dim=16, precondition_frequency=2,
                              grafting=P.GraftKind.ADAGRAD, epsilon=1e-10)
        ref = P.Shampoo([torch.tensor(p, dtype=dtype, device=cuda_device) for p in params], cfg)
        opt = P.Shampoo([torch.tensor(p, dtype=dtype, device=cuda_device) for p in params], cfg)
        lib = N.lib()
        for g in grads:
            gt = [torch.tensor(x, dtype=dtype, device=cuda_device) for x in g]
            ref.step(gt)
            t = opt.step_count
            opt.compute_directions(gt, t)  # stats + root inverse + precondition/graft
            s = torch.cuda.current_stream(cuda_device).cuda_stream
            N.check(lib.shampoo_allgather(opt._ctx, comm, C.c_void_p(s)), "allgather")
            opt.apply_gathered(t)
            opt.advance_step()
        torch.cuda.synchronize()
        for a, b in zip(ref.params(), opt.params()):
            assert torch.equal(a, b)
    finally:
        nccl.ncclCommDestroy(comm)


def test_allgather_rejects_null_comm(cuda_device):
    opt = P.Shampoo([torch.zeros(4, 4, dtype=torch.float64, device=cuda_device)])
    rc = N.lib().shampoo_allgather(opt._ctx, None, None)
    assert rc == N.ERR_INVALID_ARGUMENT
