"""B200-native Distributed Shampoo optimizer step (arXiv 2309.06497).

Drop-in for the reference's optimizer path (``minishampoo``): the same
``ShampooConfig`` / ``Shampoo`` / planning / assignment API, plus the paper's
``DistributedShampoo`` torch.optim facade.  All arithmetic of the step runs in
hand-written sm_100a kernels in ``libshampoo_b200.so`` (see include/shampoo_b200.h).
"""

from .config import (BufferOverflowError, DivergedReplicasError, GraftKind, InvalidGroupSizeError,
                     LargeDimMethod, NativeError, NonFiniteGradientError, OutOfRangeError, ShampooConfig,
                     Solver, lr_at)
from .checkpoint import CheckpointError, load_checkpoint, merge_state_trees, save_checkpoint
from .planning import (AssignmentPlan, BlockPlan, BlockRegion, BlockSpec, CommReport, GlobalBlock, NativePlan,
                       block_partition, buffer_size, comm_meter, enumerate_blocks, greedy_assign, merge_dims,
                       mlp_param_shapes, plan_parameter, plan_report, state_scalar_count)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-dependent pieces load lazily so planning works without CUDA initialisation
    if name in ("Shampoo", "GuardStats", "batched_root_inverse", "launch_count", "tc_gemm"):
        from . import optimizer
        return getattr(optimizer, name)
    if name in ("DistributedShampoo", "GroupExchange"):
        from . import distributed
        return getattr(distributed, name)
    raise AttributeError(name)


__all__ = [
    "AssignmentPlan", "BlockPlan", "CheckpointError", "load_checkpoint", "merge_state_trees", "save_checkpoint", "BlockRegion", "BlockSpec", "BufferOverflowError", "CommReport",
    "DistributedShampoo",
    "DivergedReplicasError", "GlobalBlock", "GraftKind", "GroupExchange", "GuardStats",
    "InvalidGroupSizeError", "LargeDimMethod", "NativeError", "NativePlan", "NonFiniteGradientError",
    "OutOfRangeError", "Shampoo", "ShampooConfig", "Solver", "batched_root_inverse", "tc_gemm", "block_partition",
    "buffer_size", "comm_meter", "enumerate_blocks", "greedy_assign", "launch_count", "lr_at", "merge_dims",
    "plan_parameter", "state_scalar_count",
]
