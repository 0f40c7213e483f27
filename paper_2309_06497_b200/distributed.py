"""``DistributedShampoo``: the torch.optim facade over the device-native step.

Paper API (arXiv 2309.06497 §5): ``DistributedShampoo(params,
lr, betas, epsilon, momentum, use_nesterov, weight_decay,
use_decoupled_weight_decay, use_bias_correction, max_preconditioner_dim,
precondition_frequency, start_preconditioning_step, exponent_override,
exponent_multiplier, grafting, grafting_epsilon, grafting_beta2, solver,
newton_tolerance, num_trainers_per_group)``; kwargs map 1:1 onto
``ShampooConfig`` (optim.py:53-84) and reuse its validation.

Distribution (dist.py:133-369): one process per GPU.  The
greedy plan is computed identically on every rank by the C++ planner; each
rank keeps state only for the blocks its group rank owns, writes their
directions into its region of the padded gather buffer, and an in-place NCCL
all-gather inside each group of ``num_trainers_per_group`` ranks replicates
all directions before every rank applies every block.  Groups are exact
replicas (the assignment is replicated across groups); the optional replica
check (dist.py:361-368) raises ``DivergedReplicasError`` when they are not.
"""

from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist

from .config import DivergedReplicasError, GraftKind, LargeDimMethod, ShampooConfig, Solver, lr_at
from .optimizer import GuardStats, Shampoo

__all__ = ["DistributedShampoo", "GroupExchange", "REPLICA_TOLERANCE"]

REPLICA_TOLERANCE = 1e-12  # dist.py:53


class GroupExchange:
    """Replica groups of ``group_size`` consecutive ranks and the region all-gather.

    Mirrors dist.py:350-359: every group gathers independently; group g holds
    group-local ranks [g*J_G, (g+1)*J_G) of ``process_group`` (default: WORLD).
    ``__call__(buf, group_rank, max_payload)`` fills ``buf`` (group_size *
    max_payload scalars) from every rank's region.  Backends without CUDA
    collectives (gloo with device tensors, used by the one-GPU multi-process
    tests) are served through a host staging copy.
    """

    def __init__(self, group_size: int, process_group=None):
        self.pg = process_group
        self.world = dist.get_world_size(process_group)
        self.rank = dist.get_rank(process_group)
        # new_group() takes GLOBAL ranks: map the group-local indices through the process group
        gl = (dist.get_process_group_ranks(process_group) if process_group is not None
              else list(range(self.world)))
        if group_size <= 0:
            group_size = self.world
        if self.world % group_size:
            from .config import InvalidGroupSizeError
            raise InvalidGroupSizeError(f"group size {group_size} must divide world size {self.world}")
        self.group_size = group_size
        self.group = None
        if group_size == self.world:
            self.group = process_group
        else:
            for g in range(self.world // group_size):  # every rank creates every group
                ranks = list(range(g * group_size, (g + 1) * group_size))
                pg = dist.new_group([gl[r] for r in ranks])
                if self.rank in ranks:
                    self.group = pg
        self.bytes_per_step = 0
        # cross-group communicators: ranks with the same group rank in every replica group
        self.cross = None
        if self.world // group_size > 1:
            for k in range(group_size):
                ranks = list(range(k, self.world, group_size))
                pg = dist.new_group([gl[r] for r in ranks])
                if self.rank in ranks:
                    self.cross = pg
        self.backend = dist.get_backend(process_group)
        self.staged = self.backend == "gloo"

    # -- helpers

    def _stage(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if (self.staged and t.is_cuda) else t

    def _unstage(self, host: torch.Tensor, t: torch.Tensor) -> None:
        if host is not t:
            t.copy_(host)

    # -- collectives of the step

    def reduce_gradients(self, buf: torch.Tensor, group_rank: int, max_payload: int) -> None:
        """Sum every rank's packed local gradients into the owner's region:
        reduce-scatter inside the group, then all-reduce the region across the replica groups
        (ranks holding the same blocks).  Half the bytes of a full gradient all-reduce."""
        if max_payload == 0:
            return
        full = buf[: self.group_size * max_payload]
        region = buf[group_rank * max_payload:(group_rank + 1) * max_payload]
        if self.group_size > 1:
            if self.staged:  # gloo: no reduce_scatter; all-reduce the whole group layout
                h = self._stage(full)
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.group)
                self._unstage(h, full)
            else:
                dist.reduce_scatter_tensor(region, full, op=dist.ReduceOp.SUM, group=self.group)  # in place
        if self.cross is not None:
            h = self._stage(region)
            dist.all_reduce(h, op=dist.ReduceOp.SUM, group=self.cross)
            self._unstage(h, region)

    def max_flag(self, flag: torch.Tensor) -> None:
        """Max over the optimizer's ranks of a device flag (non-finite gradient anywhere aborts everywhere)."""
        h = self._stage(flag)
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=self.pg)
        self._unstage(h, flag)

    def __call__(self, buf: torch.Tensor, group_rank: int, max_payload: int) -> None:
        if max_payload == 0 or self.group_size == 1:
            return
        region = buf[group_rank * max_payload:(group_rank + 1) * max_payload]
        out = buf[: self.group_size * max_payload]
        if self.staged:
            # gloo: list all-gather of host copies (same bytes)
            hr = region.cpu()
            parts = [torch.empty_like(hr) for _ in range(self.group_size)]
            dist.all_gather(parts, hr, group=self.group)
            out.copy_(torch.cat(parts).to(out.device))
        else:
            dist.all_gather_into_tensor(out, region, group=self.group)  # in place (NCCL)
        self.bytes_per_step = (self.group_size - 1) * max_payload * buf.element_size()

    def gather_group_trees(self, tree: dict) -> list:
        """Every rank's state tree of this rank's replica group (host objects), in group-rank order."""
        out = [None] * self.group_size
        if self.group_size == 1:
            return [tree]
        dist.all_gather_object(out, tree, group=self.group)
        return out

    def check_replicas(self, params, tolerance: float = REPLICA_TOLERANCE) -> float:
        """dist.py:361-368: every rank's parameters must match to ``tolerance`` (max abs).  Exact
        elementwise check: all-reduce MAX and MIN of the flat float64 parameters over all ranks;
        raises DivergedReplicasError with the largest drift.  Costs two all-reduces of the
        parameters, so the optimizer runs it only every ``check_replicas_every`` steps."""
        flat = torch.cat([p.detach().reshape(-1).to(torch.float64) for p in params]) if params else None
        if flat is None or flat.numel() == 0:
            return 0.0
        hi, lo = self._stage(flat.clone()), self._stage(flat.clone())
        dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=self.pg)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=self.pg)
        drift = float((hi - lo).abs().max().item())
        if not drift <= tolerance:
            raise DivergedReplicasError(f"replicas drifted {drift:.3e} (max over ranks) > {tolerance:g}")
        return drift


class DistributedShampoo(torch.optim.Optimizer):
    """Drop-in ``torch.optim.Optimizer`` running the B200 Shampoo step.

    ``step()`` reads ``p.grad`` and updates ``p`` in place.  Learning rate: with the constant
    schedule the param group's ``lr`` is used every step (so torch LR schedulers work); with
    ``lr_schedule="warmup_cosine"`` the schedule lr_at(t) (optim.py:133-151) is scaled by
    ``param_groups[0]['lr'] / lr``.  Parameters whose ``grad`` is None take a zero gradient: their
    blocks still receive the decoupled weight decay, momentum and factor decay of a zero-gradient
    step (the reference step requires a gradient for every parameter, optim.py:358-374).
    """

    def __init__(self, params, lr: float = 0.1, betas=(0.0, 0.999), epsilon: float = 1e-12,
                 momentum: float = 0.9, use_nesterov: bool = True, weight_decay: float = 1e-4,
                 use_decoupled_weight_decay: bool = True, use_bias_correction: bool = True,
                 max_preconditioner_dim: int = 2048, precondition_frequency: int = 50,
                 start_preconditioning_step: float = 0, exponent_override: int = 0,
                 exponent_multiplier: float = 1.0, grafting=GraftKind.SGD,
                 grafting_epsilon: float = 1e-8, grafting_beta2: float = 0.999, solver=Solver.EIGH,
                 newton_tolerance: float = 1e-6, num_trainers_per_group: int = -1,
                 large_dim_method=LargeDimMethod.BLOCKING, precision: str = "double",
                 lr_schedule: str = "constant", warmup_steps: int = 0, total_steps: int = 0,
                 process_group=None, reduce_gradients: Optional[str] = None,
                 check_replicas_every: int = 0, check_finite=True):
        """``reduce_gradients``: None (p.grad already holds the global gradient, e.g. after DDP) or
        "mean" / "sum": p.grad holds this rank's LOCAL gradient and the optimizer reduce-scatters
        it to the block owners itself (no separate DDP all-reduce needed).
        ``check_replicas_every``: run the replica drift check (dist.py:361-368) every N steps (0: off).
        ``check_finite``: True (raise from the bad step, one host sync per step), "deferred" (no host
        sync; the bad step is skipped on the device and the next call raises), False."""
        if reduce_gradients not in (None, "mean", "sum"):
            raise ValueError("reduce_gradients must be None, 'mean' or 'sum'")
        if check_replicas_every < 0:
            raise ValueError("check_replicas_every must be non-negative")
        self.reduce_gradients = reduce_gradients
        self.check_replicas_every = int(check_replicas_every)
        grafting = GraftKind(grafting) if not isinstance(grafting, GraftKind) else grafting
        solver = Solver(solver) if not isinstance(solver, Solver) else solver
        large_dim_method = (LargeDimMethod(large_dim_method)
                            if not isinstance(large_dim_method, LargeDimMethod) else large_dim_method)
        self.config = ShampooConfig(
            lr=lr, lr_schedule=lr_schedule, warmup_steps=warmup_steps, total_steps=total_steps,
            betas=tuple(betas), epsilon=epsilon, momentum=momentum, use_nesterov=use_nesterov,
            weight_decay=weight_decay, use_decoupled_weight_decay=use_decoupled_weight_decay,
            use_bias_correction=use_bias_correction, max_preconditioner_dim=max_preconditioner_dim,
            precondition_frequency=precondition_frequency,
            start_preconditioning_step=start_preconditioning_step, exponent_override=exponent_override,
            exponent_multiplier=exponent_multiplier, grafting=grafting, grafting_epsilon=grafting_epsilon,
            grafting_beta2=grafting_beta2, large_dim_method=large_dim_method, solver=solver,
            newton_tolerance=newton_tolerance, precision=precision)
        defaults = dict(lr=lr, betas=tuple(betas), epsilon=epsilon, momentum=momentum,
                        weight_decay=weight_decay)
        super().__init__(params, defaults)
        if len(self.param_groups) != 1:
            raise ValueError("DistributedShampoo supports a single parameter group")
        self._plist = list(self.param_groups[0]["params"])
        if dist.is_available() and dist.is_initialized():
            self.exchange = GroupExchange(num_trainers_per_group, process_group)
            world, rank, group = self.exchange.world, self.exchange.rank, self.exchange.group_size
        else:
            if num_trainers_per_group not in (-1, 0, 1):
                raise ValueError("num_trainers_per_group > 1 needs torch.distributed to be initialised")
            self.exchange, world, rank, group = None, 1, 0, 1
        self.engine = Shampoo([p.data for p in self._plist], self.config, world_size=world,
                              group_size=group, rank=rank, exchange=self.exchange, check_finite=check_finite)

    @property
    def guard_stats(self) -> GuardStats:
        return self.engine.guard_stats

    @property
    def step_count(self) -> int:
        return self.engine.step_count

    def current_lr(self) -> float:
        """The learning rate the next step applies (see the class docstring)."""
        group_lr = float(self.param_groups[0]["lr"])
        if self.config.lr_schedule == "constant":
            return group_lr
        return lr_at(self.config, self.engine.step_count) * (group_lr / self.config.lr)

    @torch.no_grad()
    def step(self, closure=None):
        loss = None
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        grads = [p.grad if p.grad is not None else torch.zeros_like(p) for p in self._plist]
        lr = self.current_lr()
        if self.reduce_gradients is None:
            self.engine.step(grads, lr=lr)
        else:
            self.engine.step_local(grads, average=self.reduce_gradients == "mean", lr=lr)
        if (self.exchange is not None and self.check_replicas_every
                and self.engine.step_count % self.check_replicas_every == 0):
            self.exchange.check_replicas(self._plist)
        return loss

    def state_dict(self) -> dict:
        """``state_tree`` nesting (optim.py:387-423) plus the torch param-group metadata."""
        return {"state": self.engine.state_tree(), "param_groups": [
            {k: v for k, v in g.items() if k != "params"} for g in self.param_groups]}

    def full_state_tree(self) -> dict:
        """The union of the replica group's per-rank trees (train.py:346-353): every block once."""
        from .checkpoint import merge_state_trees
        tree = self.engine.state_tree()
        if self.exchange is None:
            return tree
        return merge_state_trees(self.exchange.gather_group_trees(tree))

    def save_checkpoint(self, path: str) -> None:
        """Reference-format checkpoint of the whole optimizer (checkpoint.py:114-126): the sharded
        state is merged across the replica group; rank 0 writes the file (collective call)."""
        from .checkpoint import save_checkpoint
        tree = self.full_state_tree()
        if self.exchange is None or self.exchange.rank == 0:
            save_checkpoint(path, self.engine.step_count, [p.detach().cpu().numpy() for p in self._plist], tree)

    def load_checkpoint(self, path: str) -> None:
        """Resume from a reference-format checkpoint (each rank loads its owned blocks)."""
        self.engine.load_checkpoint(path)

    def load_state_dict(self, state_dict: dict) -> None:
        self.engine.load_state_tree(state_dict["state"])
        for g, saved in zip(self.param_groups, state_dict.get("param_groups", [])):
            for k, v in saved.items():
                if k != "params":
                    g[k] = v
