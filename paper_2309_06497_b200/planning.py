"""Block planning and block-to-rank assignment (host mirror over the C++ planner).

Same names and semantics as the reference:
  merge_dims            precond.py:56-77
  BlockSpec / block_partition / plan_parameter   precond.py:80-158
  GlobalBlock / enumerate_blocks                 dist.py:77-86, 232-243
  BlockRegion / AssignmentPlan / greedy_assign / buffer_size   dist.py:68-183
The integer work runs in ``csrc/planner.cpp`` (bit-exact with the reference);
this module only marshals it.  Offsets: ``BlockRegion.byte_offset`` keeps the
reference's 8-byte-scalar convention (dist.py:48-50) so plans compare 1:1;
``scalar_offset`` is what the device gather buffer uses.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from itertools import product
from typing import Optional, Sequence

from . import _native as N
from .config import LargeDimMethod, METHOD_CODES

__all__ = [
    "SCALAR_BYTES", "merge_dims", "BlockSpec", "BlockPlan", "block_partition", "plan_parameter",
    "GlobalBlock", "BlockRegion", "AssignmentPlan", "NativePlan", "enumerate_blocks", "greedy_assign",
    "buffer_size", "state_scalar_count", "CommReport", "comm_meter",
]

SCALAR_BYTES = 8  # reference wire scalar (dist.py:48-50)
_METHODS = {v: k for k, v in METHOD_CODES.items()}


def merge_dims(shape: Sequence[int], max_dim: int) -> tuple[int, ...]:
    shape = tuple(int(d) for d in shape)
    arr = (C.c_int64 * max(len(shape), 1))(*shape)
    out = (C.c_int64 * max(len(shape), 1))()
    nd = C.c_int32()
    N.check(N.lib().shampoo_merge_dims(arr, len(shape), int(max_dim), out, C.byref(nd)), "merge_dims")
    return tuple(out[i] for i in range(nd.value))


@dataclass(frozen=True)
class BlockSpec:
    ranges: tuple[tuple[int, int], ...]

    @property
    def shape(self) -> tuple[int, ...]:
        return tuple(hi - lo for lo, hi in self.ranges)

    @property
    def var_count(self) -> int:
        return math.prod(self.shape)

    @property
    def slices(self) -> tuple[slice, ...]:
        return tuple(slice(lo, hi) for lo, hi in self.ranges)


def block_partition(shape: Sequence[int], block_size: int) -> tuple[BlockSpec, ...]:
    """ceil(d/b) ranges per dim, row-major (precond.py:99-111); host-side helper."""
    if block_size < 1:
        raise ValueError("block_size must be at least 1")
    cuts = [[(lo, min(lo + block_size, d)) for lo in range(0, d, block_size)] for d in shape]
    return tuple(BlockSpec(ranges=c) for c in product(*cuts))


@dataclass(frozen=True)
class BlockPlan:
    original_shape: tuple[int, ...]
    merged_shape: tuple[int, ...]
    block_size: int
    method: LargeDimMethod
    blocks: tuple[BlockSpec, ...]

    @property
    def block_shapes(self):
        return tuple(b.shape for b in self.blocks)


@dataclass(frozen=True)
class GlobalBlock:
    block_id: int
    param_index: int
    block_index: int
    var_count: int
    shape: tuple[int, ...]


@dataclass(frozen=True)
class BlockRegion:
    owner_rank: int
    byte_offset: int
    byte_length: int

    @property
    def scalar_offset(self) -> int:
        return self.byte_offset // SCALAR_BYTES


class NativePlan:
    """Owns a ``shampoo_plan*``: planning for a list of parameter shapes."""

    def __init__(self, shapes: Sequence[Sequence[int]], max_dim: int,
                 method: LargeDimMethod = LargeDimMethod.BLOCKING, world_size: int = 1,
                 group_size: int = 1):
        shapes = [tuple(int(d) for d in s) for s in shapes]
        flat = [d for s in shapes for d in s]
        arr = (C.c_int64 * max(len(flat), 1))(*flat)
        nd = (C.c_int32 * max(len(shapes), 1))(*[len(s) for s in shapes])
        h = C.c_void_p()
        N.check(N.lib().shampoo_plan_create(arr, nd, len(shapes), int(max_dim), METHOD_CODES[method],
                                            int(world_size), int(group_size), C.byref(h)), "plan_create")
        self.handle = h
        self.shapes = shapes
        self.max_dim = int(max_dim)
        self.world_size = int(world_size)
        self.group_size = int(group_size)
        lib = N.lib()
        self.blocks_info: list[N.BlockInfo] = []
        for i in range(lib.shampoo_plan_num_blocks(h)):
            info = N.BlockInfo()
            N.check(lib.shampoo_plan_block(h, i, C.byref(info)), "plan_block")
            self.blocks_info.append(info)
        self.param_plans: list[BlockPlan] = []
        per_param: dict[int, list[BlockSpec]] = {}
        for info in self.blocks_info:
            per_param.setdefault(info.param_index, []).append(
                BlockSpec(tuple((info.lo[k], info.hi[k]) for k in range(info.order))))
        for p, s in enumerate(shapes):
            merged = (C.c_int64 * N.MAX_ORDER)()
            mnd, meth = C.c_int32(), C.c_int32()
            N.check(lib.shampoo_plan_param(h, p, merged, C.byref(mnd), C.byref(meth)), "plan_param")
            self.param_plans.append(BlockPlan(s, tuple(merged[k] for k in range(mnd.value)), self.max_dim,
                                              _METHODS[meth.value], tuple(per_param.get(p, ()))))
        counters = (C.c_int64 * self.group_size)()
        lib.shampoo_plan_counters(h, counters)
        self.counters = tuple(counters)
        self.max_payload = int(lib.shampoo_plan_max_payload(h))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                N.lib().shampoo_plan_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def global_blocks(self) -> tuple[GlobalBlock, ...]:
        return tuple(GlobalBlock(b.block_id, b.param_index, b.block_index, b.var_count,
                                 tuple(b.hi[k] - b.lo[k] for k in range(b.order)))
                     for b in self.blocks_info)

    def owned_ids(self, rank: int) -> frozenset[int]:
        k = rank % self.group_size
        return frozenset(b.block_id for b in self.blocks_info if b.owner_rank == k)


def plan_parameter(shape: Sequence[int], max_dim: int,
                   configured: LargeDimMethod = LargeDimMethod.BLOCKING) -> BlockPlan:
    return NativePlan([shape], max_dim, configured).param_plans[0]


def enumerate_blocks(param_shapes: Sequence[Sequence[int]], config) -> tuple[GlobalBlock, ...]:
    return NativePlan(param_shapes, config.max_preconditioner_dim, config.large_dim_method).global_blocks


@dataclass(frozen=True)
class AssignmentPlan:
    """dist.py:88-130 (offsets in reference 8-byte scalars)."""

    world_size: int
    group_size: int
    assignments: tuple[frozenset[int], ...]
    counters: tuple[int, ...]
    buffer_layout: dict
    var_counts: tuple[int, ...]

    @property
    def num_groups(self) -> int:
        return self.world_size // self.group_size

    @property
    def max_payload_bytes(self) -> int:
        return max(self.counters) * SCALAR_BYTES

    def owned_by_group_rank(self, k: int) -> frozenset[int]:
        return self.assignments[k]

    def to_json_dict(self) -> dict:
        return {
            "world_size": self.world_size, "group_size": self.group_size, "num_groups": self.num_groups,
            "counters": list(self.counters), "buffer_bytes": buffer_size(self),
            "assignments": [sorted(a) for a in self.assignments],
            "blocks": {str(i): {"owner_rank": r.owner_rank, "byte_offset": r.byte_offset,
                                "byte_length": r.byte_length} for i, r in sorted(self.buffer_layout.items())},
        }


def _assignment_from_native(np_: NativePlan) -> AssignmentPlan:
    owned = [set() for _ in range(np_.group_size)]
    layout = {}
    for b in np_.blocks_info:
        owned[b.owner_rank].add(b.block_id)
        layout[b.block_id] = BlockRegion(b.owner_rank, b.gather_offset * SCALAR_BYTES, b.var_count * SCALAR_BYTES)
    return AssignmentPlan(np_.world_size, np_.group_size,
                          tuple(frozenset(owned[r % np_.group_size]) for r in range(np_.world_size)),
                          np_.counters, layout, tuple(b.var_count for b in np_.blocks_info))


def greedy_assign(block_var_counts: Sequence[int], world_size: int, group_size: int) -> AssignmentPlan:
    """Algorithm 3 (dist.py:133-176) through the C++ planner: each count is fed
    as a 1-D parameter of that length with max_dim >= every count, so each
    becomes exactly one block."""
    counts = [int(c) for c in block_var_counts]
    if any(c <= 0 for c in counts):
        raise ValueError("block variable counts must be positive")
    np_ = NativePlan([(c,) for c in counts], max(counts) if counts else 1, LargeDimMethod.BLOCKING,
                     world_size, group_size)
    return _assignment_from_native(np_)


def assignment_for(np_: NativePlan) -> AssignmentPlan:
    return _assignment_from_native(np_)


def buffer_size(plan: AssignmentPlan) -> int:
    """Bytes of the flat gather buffer in the reference's 8-byte wire format (dist.py:179-183)."""
    if not plan.var_counts:
        return 0
    return plan.group_size * plan.max_payload_bytes


def state_scalar_count(shape: tuple[int, ...], method: LargeDimMethod) -> int:
    """precond.py:399-410."""
    if method is LargeDimMethod.BLOCKING:
        return 2 * sum(d * d for d in shape)
    if method is LargeDimMethod.ADAGRAD:
        return math.prod(shape)
    return sum(shape)


@dataclass(frozen=True)
class CommReport:
    """Deterministic communication and memory accounting for a plan (dist.py:370-391)."""

    steps: int
    bytes_gathered_per_step: int  # one group's buffer, per step
    world_bytes_per_step: int  # all replica groups together
    total_bytes_gathered: int
    per_worker_state_scalars: tuple
    per_worker_state_bytes: tuple

    def to_json_dict(self) -> dict:
        return {
            "steps": self.steps,
            "bytes_gathered_per_step": self.bytes_gathered_per_step,
            "world_bytes_per_step": self.world_bytes_per_step,
            "total_bytes_gathered": self.total_bytes_gathered,
            "per_worker_state_scalars": list(self.per_worker_state_scalars),
            "per_worker_state_bytes": list(self.per_worker_state_bytes),
        }


def comm_meter(plan: AssignmentPlan, block_shapes: Sequence[Sequence[int]],
               method: LargeDimMethod = LargeDimMethod.BLOCKING, steps: int = 1) -> CommReport:
    """Gathered bytes per step and per-worker state footprint (dist.py:394-423), in the
    reference's 8-byte wire scalars (the device buffer uses the context's element size)."""
    if len(block_shapes) != len(plan.var_counts):
        raise ValueError("one shape per planned block required")
    per_group = buffer_size(plan)
    world = per_group * plan.num_groups
    state = tuple(sum(state_scalar_count(tuple(block_shapes[i]), method) for i in plan.assignments[r])
                  for r in range(plan.world_size))
    return CommReport(steps=steps, bytes_gathered_per_step=per_group, world_bytes_per_step=world,
                      total_bytes_gathered=world * steps, per_worker_state_scalars=state,
                      per_worker_state_bytes=tuple(x * SCALAR_BYTES for x in state))


def plan_report(param_shapes: Sequence[Sequence[int]], config, world_size: int = 1,
                group_size: Optional[int] = None, steps: int = 100) -> dict:
    """The JSON document of the reference's ``minishampoo plan`` command (cli.py:168-218):
    the assignment plan, its communication report and per-parameter state accounting for every
    large-dimension method.  ``param_shapes`` in the reference trainer's (d_out, d_in) layout
    for MLP widths (cli.py:172); ``group_size`` None = the whole world (num_trainers_per_group -1)."""
    group = world_size if group_size is None else int(group_size)
    blocks = enumerate_blocks(param_shapes, config)
    plan = greedy_assign([b.var_count for b in blocks], world_size, group)
    report = comm_meter(plan, [b.shape for b in blocks], method=config.large_dim_method, steps=steps)
    per_parameter = []
    for shape in param_shapes:
        methods = {}
        for method in LargeDimMethod:
            pp = plan_parameter(shape, config.max_preconditioner_dim, method)
            methods[method.value] = sum(state_scalar_count(spec.shape, method) for spec in pp.blocks)
        pp = plan_parameter(shape, config.max_preconditioner_dim, config.large_dim_method)
        per_parameter.append({"shape": list(shape), "merged_shape": list(pp.merged_shape),
                              "num_blocks": len(pp.blocks), "state_scalars_by_method": methods})
    return {"plan": plan.to_json_dict(), "comm": report.to_json_dict(), "per_parameter": per_parameter}


def mlp_param_shapes(widths: Sequence[int]) -> list[tuple[int, int]]:
    """Weight shapes of the reference trainer's MLP: (d_out, d_in) per layer (cli.py:172, train.py:93)."""
    return [(d_out, d_in) for d_in, d_out in zip(widths, widths[1:])]
