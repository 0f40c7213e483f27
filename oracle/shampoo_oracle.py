"""CPU oracle for the Distributed Shampoo optimizer step -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference package
``minishampoo`` (``/root/reference/pkg/src/minishampoo``) for the one hot path
this repository accelerates: the optimizer step (planning, factor statistics,
root inverse, grafting, momentum, sharded gather, parameter update).

It exists to CHECK the B200 implementation, never to stand in for it:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
(``paper_2309_06497_b200``) must not import this file.

Parity pinning: the oracle is checked against (a) the reference's own golden
known-answer tests, restated in ``tests/test_oracle_golden.py``, and (b)
fixtures produced by running the real reference in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), compared in
``tests/test_oracle_fixtures.py``.  Parity is therefore PINNED.

Citations are ``file:line`` relative to ``/root/reference/pkg/src/minishampoo``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from itertools import product
from typing import Sequence

import numpy as np

SCALAR_BYTES = 8  # dist.py:48-50 (one LE float64 per direction scalar)
SYMMETRY_RTOL = 1e-12  # matfun.py:32
NEWTON_DEFAULT_TOL = 1e-6  # matfun.py:34
NEWTON_MAX_ITERATIONS = 1000  # matfun.py:35


class GraftKind(Enum):  # grafting.py:18-25
    SGD = "sgd"
    ADAGRAD = "adagrad"
    RMSPROP = "rmsprop"
    ADAM = "adam"
    NORMALIZED_ADAGRAD = "normalized_adagrad"
    NORMALIZED_RMSPROP = "normalized_rmsprop"
    NORMALIZED_ADAM = "normalized_adam"


class Solver(Enum):  # matfun.py:50-52
    EIGH = "eigh"
    COUPLED_NEWTON = "newton"


class LargeDimMethod(Enum):  # precond.py:50-53
    BLOCKING = "blocking"
    ADAGRAD = "adagrad"
    DIAGONAL = "diagonal"


class OracleSolverFailure(Exception):
    """Recoverable root-inverse failure (matfun.py:254-259 'recoverable' set)."""


# ---------------------------------------------------------------- planning


def merge_dims(shape: Sequence[int], max_dim: int) -> tuple[int, ...]:
    """Greedy left-to-right fold while the running product stays <= max_dim.

    precond.py:56-77: size-1 dims always fold, an oversize dim is kept, an
    empty/all-ones shape becomes (1,).
    """
    if max_dim < 1:
        raise ValueError("max_dim must be at least 1")
    out: list[int] = []
    acc = 1
    for d in shape:
        if d < 1:
            raise ValueError(f"dimensions must be positive, got {tuple(shape)}")
        if acc == 1 or d == 1 or acc * d <= max_dim:
            acc *= d
        else:
            out.append(acc)
            acc = d
    if acc > 1 or not out:
        out.append(acc)
    return tuple(out)


def block_ranges(shape: Sequence[int], b: int) -> list[tuple[tuple[int, int], ...]]:
    """ceil(d/b) half-open cuts per dim, enumerated row-major (precond.py:99-111)."""
    if b < 1:
        raise ValueError("block_size must be at least 1")
    cuts = [[(lo, min(lo + b, d)) for lo in range(0, d, b)] for d in shape]
    return [tuple(c) for c in product(*cuts)]


def plan_parameter(shape: Sequence[int], max_dim: int,
                   method: LargeDimMethod = LargeDimMethod.BLOCKING):
    """(merged_shape, effective_method, ranges) -- precond.py:114-158."""
    merged = merge_dims(tuple(shape), max_dim)
    if all(d <= max_dim for d in merged):
        method = LargeDimMethod.BLOCKING
    if method is LargeDimMethod.BLOCKING:
        ranges = block_ranges(merged, max_dim)
    else:
        ranges = [tuple((0, d) for d in merged)]
    return merged, method, ranges


@dataclass(frozen=True)
class OracleBlock:
    block_id: int
    param_index: int
    block_index: int
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


def enumerate_blocks(shapes: Sequence[Sequence[int]], max_dim: int,
                     method: LargeDimMethod = LargeDimMethod.BLOCKING):
    """Param-major, block-minor global ids (dist.py:232-243)."""
    blocks = []
    for i, s in enumerate(shapes):
        _, _, ranges = plan_parameter(s, max_dim, method)
        for b, r in enumerate(ranges):
            blocks.append(OracleBlock(len(blocks), i, b, r))
    return blocks


@dataclass
class OracleAssignment:
    world_size: int
    group_size: int
    owner: list[int]  # group rank per block id
    counters: list[int]
    offsets: list[int]  # absolute scalar offset of each block in the gather buffer
    var_counts: list[int]

    @property
    def max_payload(self) -> int:
        return max(self.counters) if self.var_counts else 0

    def owned(self, rank: int) -> list[int]:
        k = rank % self.group_size
        return sorted(i for i, o in enumerate(self.owner) if o == k)

    @property
    def buffer_scalars(self) -> int:
        return self.group_size * self.max_payload if self.var_counts else 0


def greedy_assign(var_counts: Sequence[int], world_size: int, group_size: int) -> OracleAssignment:
    """Algorithm 3 / dist.py:133-176: LPT greedy + padded rank-region layout."""
    if world_size < 1 or group_size < 1 or world_size % group_size:
        raise ValueError(f"group size {group_size} must divide world size {world_size}")
    counts = [int(c) for c in var_counts]
    if any(c <= 0 for c in counts):
        raise ValueError("block variable counts must be positive")
    load = [0] * group_size
    owner = [-1] * len(counts)
    for i in sorted(range(len(counts)), key=lambda j: (-counts[j], j)):
        k = min(range(group_size), key=lambda r: (load[r], r))
        owner[i] = k
        load[k] += counts[i]
    width = max(load) if counts else 0
    offsets = [0] * len(counts)
    for k in range(group_size):
        at = k * width
        for i in range(len(counts)):
            if owner[i] == k:
                offsets[i] = at
                at += counts[i]
    return OracleAssignment(world_size, group_size, owner, load, offsets, counts)


# ---------------------------------------------------------------- linear algebra


def mode_gram(g: np.ndarray, k: int) -> np.ndarray:
    """Symmetrised mode-k contraction of g with itself (precond.py:161-165)."""
    other = [a for a in range(g.ndim) if a != k]
    c = np.tensordot(g, g, axes=(other, other))
    return (c + c.T) / 2


def mode_apply(m: np.ndarray, g: np.ndarray, k: int) -> np.ndarray:
    """refold(m @ unfold_k(g)) (precond.py:168-174)."""
    return np.moveaxis(np.tensordot(m, g, axes=(1, k)), 0, k)


def _validate(a: np.ndarray) -> np.ndarray:
    """matfun.py:108-118: square, finite (recoverable), symmetric (NOT recoverable)."""
    a = np.asarray(a)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("expected a square matrix")
    if not np.all(np.isfinite(a)):
        raise OracleSolverFailure("non-finite input")
    if np.linalg.norm(a - a.T) > SYMMETRY_RTOL * max(float(np.linalg.norm(a)), 1.0):
        raise ValueError("matrix is not symmetric")
    return a


def root_inverse_eigh(a: np.ndarray, p: int, eta: float = 1.0, eps: float = 0.0) -> np.ndarray:
    """Spectral A^(-eta/p) with the shift-clamp w - min(w_min,0) + eps (matfun.py:139-157)."""
    a = _validate(a)
    try:
        w, q = np.linalg.eigh(a)
    except np.linalg.LinAlgError as exc:  # matfun.py:134-135
        raise OracleSolverFailure(str(exc)) from exc
    shift = min(float(w.min()), 0.0) if w.size else 0.0
    w = w - shift + eps
    if eps == 0.0 and np.any(w <= 0.0):
        raise OracleSolverFailure("epsilon zero with singular matrix")
    with np.errstate(over="ignore", divide="ignore", invalid="ignore"):
        x = (q * w ** (-eta / p)) @ q.T
    return (x + x.T) / 2


def root_inverse_newton(a: np.ndarray, p: int, eps: float = 0.0,
                        tol: float = NEWTON_DEFAULT_TOL):
    """Coupled inverse Newton (matfun.py:164-222). Returns (x, iters, residual, converged)."""
    a = _validate(a)
    n = a.shape[0]
    eye = np.eye(n, dtype=a.dtype)
    if float(np.linalg.norm(a)) == 0.0:
        if eps == 0.0:
            raise OracleSolverFailure("zero matrix with epsilon zero")
        return eps ** (-1.0 / p) * eye, 0, 0.0, True
    if eps > 0.0:
        a = a + eps * eye
    c = float((2.0 * np.linalg.norm(a) / (p + 1)) ** (1.0 / p))
    x = eye / c
    m = a / c ** p
    best, best_res, it, ok = x, math.inf, 0, False
    with np.errstate(over="ignore", invalid="ignore"):
        for it in range(1, NEWTON_MAX_ITERATIONS + 1):
            t = ((p + 1) * eye - m) / p
            x = x @ t
            m = np.linalg.matrix_power(t, p) @ m
            res = float(np.abs(m - eye).sum(axis=1).max())
            if not np.isfinite(res):
                break
            if res < best_res:
                best, best_res = x, res
            if res < tol:
                ok = True
                break
    return (best + best.T) / 2, it, best_res, ok


@dataclass
class GuardCounts:  # matfun.py:98-105
    primary: int = 0
    double_retry: int = 0
    fallback_previous: int = 0
    fallback_identity: int = 0


def guarded_root_inverse(a, p, eta, eps, solver, tol, previous, counts: GuardCounts):
    """Requested precision -> float64 retry -> previous -> eps^(-eta/p) I (matfun.py:240-293)."""

    def attempt(m):
        if solver is Solver.COUPLED_NEWTON:
            x, _, _, ok = root_inverse_newton(m, p, eps, tol)
            if not ok:
                raise OracleSolverFailure("newton did not converge")
        else:
            x = root_inverse_eigh(m, p, eta, eps)
        if not np.all(np.isfinite(x)):
            raise OracleSolverFailure("non-finite result")
        return x

    try:
        x = attempt(a)
        counts.primary += 1
        return x
    except OracleSolverFailure:
        pass
    try:
        x = attempt(np.asarray(a, dtype=np.float64))
        counts.double_retry += 1
        return x
    except OracleSolverFailure:
        pass
    if previous is not None:
        counts.fallback_previous += 1
        return previous
    counts.fallback_identity += 1
    scale = eps ** (-eta / p) if eps > 0.0 else 1.0
    return scale * np.eye(np.asarray(a).shape[0])


# ---------------------------------------------------------------- config


@dataclass(frozen=True)
class OracleConfig:
    """Same fields and defaults as ShampooConfig (optim.py:53-84)."""

    lr: float = 0.1
    lr_schedule: str = "constant"
    warmup_steps: int = 0
    total_steps: int = 0
    betas: tuple = (0.0, 0.999)
    epsilon: float = 1e-12
    momentum: float = 0.9
    use_nesterov: bool = True
    weight_decay: float = 1e-4
    use_decoupled_weight_decay: bool = True
    use_bias_correction: bool = True
    max_preconditioner_dim: int = 2048
    precondition_frequency: int = 50
    start_preconditioning_step: float = 0
    exponent_override: int = 0
    exponent_multiplier: float = 1.0
    grafting: GraftKind = GraftKind.SGD
    grafting_epsilon: float = 1e-8
    grafting_beta2: float = 0.999
    large_dim_method: LargeDimMethod = LargeDimMethod.BLOCKING
    solver: Solver = Solver.EIGH
    newton_tolerance: float = 1e-6
    precision: str = "double"


def lr_at(cfg: OracleConfig, t: int) -> float:
    """Constant or linear-warmup + cosine (optim.py:133-151)."""
    if t < 0:
        raise ValueError("negative step")
    if cfg.lr_schedule == "constant":
        return cfg.lr
    if t >= cfg.total_steps:
        raise ValueError("step beyond total_steps")
    w = cfg.warmup_steps
    if t < w:
        return cfg.lr * (t + 1) / w
    span = cfg.total_steps - w
    if span == 0:
        return cfg.lr
    return cfg.lr * 0.5 * (1.0 + math.cos(math.pi * (t - w) / span))


# ---------------------------------------------------------------- per-block state


_NORMALIZED = {GraftKind.NORMALIZED_ADAGRAD, GraftKind.NORMALIZED_RMSPROP, GraftKind.NORMALIZED_ADAM}
_SUMMED = {GraftKind.ADAGRAD, GraftKind.NORMALIZED_ADAGRAD}
_DEBIASED = {GraftKind.ADAM, GraftKind.NORMALIZED_ADAM}


@dataclass
class OracleBlockState:
    shape: tuple
    kind: str  # shampoo | graft_only | adagrad | diagonal
    factors: list = field(default_factory=list)
    inverses: list | None = None
    step: int = 0
    last_inverse_step: int = -1
    graft_acc: np.ndarray | None = None
    graft_step: int = 0
    filtered: np.ndarray | None = None
    momentum: np.ndarray | None = None
    diag_acc: np.ndarray | None = None  # AdaGrad fallback accumulator
    diags: list | None = None  # diagonal-Shampoo per-mode vectors


class OracleShampoo:
    """Single-process Shampoo step over float64 numpy parameters.

    Follows Shampoo.step / block_direction / apply_directions (optim.py:278-383).
    ``owned`` restricts state to a set of (param, block) pairs exactly like
    the reference's sharded workers (optim.py:205-210).
    """

    def __init__(self, params, cfg: OracleConfig, owned=None):
        self.cfg = cfg
        self.t = 0
        self.guard = GuardCounts()
        self.params = [np.ascontiguousarray(np.asarray(p, dtype=np.float64)) for p in params]
        self.plans = []
        self.states: list[list[OracleBlockState | None]] = []
        fdt = np.float32 if cfg.precision == "single" else np.float64
        b1 = cfg.betas[0]
        for i, p in enumerate(self.params):
            merged, method, ranges = plan_parameter(p.shape, cfg.max_preconditioner_dim,
                                                    cfg.large_dim_method)
            self.plans.append((merged, method, ranges))
            row = []
            for b, r in enumerate(ranges):
                if owned is not None and (i, b) not in owned:
                    row.append(None)
                    continue
                shape = tuple(hi - lo for lo, hi in r)
                if all(d == 1 for d in shape):
                    kind = "graft_only"
                elif method is LargeDimMethod.BLOCKING:
                    kind = "shampoo"
                elif method is LargeDimMethod.ADAGRAD:
                    kind = "adagrad"
                else:
                    kind = "diagonal"
                st = OracleBlockState(shape, kind)
                if kind == "shampoo":
                    st.factors = [np.zeros((d, d), dtype=fdt) for d in shape]
                elif kind == "adagrad":
                    st.diag_acc = np.zeros(shape, dtype=fdt)
                elif kind == "diagonal":
                    st.diags = [np.zeros(d, dtype=fdt) for d in shape]
                if cfg.grafting is not GraftKind.SGD:
                    st.graft_acc = np.zeros(shape)
                if b1 > 0.0:
                    st.filtered = np.zeros(shape)
                if cfg.momentum > 0.0:
                    st.momentum = np.zeros(shape)
                row.append(st)
            self.states.append(row)

    # -- helpers

    def root_p(self, order: int) -> int:
        return self.cfg.exponent_override or 2 * order  # precond.py:217

    def merged(self, i):
        return self.params[i].reshape(self.plans[i][0])

    def _graft_update(self, st: OracleBlockState, g):  # grafting.py:68-83
        cfg = self.cfg
        st.graft_step += 1
        if cfg.grafting is GraftKind.SGD:
            return
        if cfg.grafting in _NORMALIZED:
            nrm = float(np.linalg.norm(g))
            if nrm > 0.0:
                g = g / nrm
        if cfg.grafting in _SUMMED:
            st.graft_acc += g * g
        else:
            st.graft_acc *= cfg.grafting_beta2
            st.graft_acc += (1.0 - cfg.grafting_beta2) * (g * g)

    def _graft_direction(self, st: OracleBlockState, g_eff):  # grafting.py:85-92
        cfg = self.cfg
        if cfg.grafting is GraftKind.SGD:
            return np.array(g_eff, dtype=np.float64, copy=True)
        acc = st.graft_acc
        if cfg.grafting in _DEBIASED and cfg.use_bias_correction and st.graft_step > 0:
            acc = acc / (1.0 - cfg.grafting_beta2 ** st.graft_step)
        return g_eff / (np.sqrt(acc) + cfg.grafting_epsilon)

    def _factor_update(self, st: OracleBlockState, g):  # precond.py:232-242
        beta2 = self.cfg.betas[1]
        for k, f in enumerate(st.factors):
            c = mode_gram(g, k).astype(f.dtype, copy=False)
            if beta2 == 1.0:
                f += c
            else:
                f *= beta2
                f += (1.0 - beta2) * c
        st.step += 1

    def _maybe_refresh(self, st: OracleBlockState, t: int):  # precond.py:244-267
        cfg = self.cfg
        if t < cfg.start_preconditioning_step or t % cfg.precondition_frequency != 0:
            return
        beta2 = cfg.betas[1]
        corr = 1.0 - beta2 ** (t + 1) if (cfg.use_bias_correction and beta2 < 1.0) else 1.0
        p = self.root_p(len(st.shape))
        new = []
        for k, f in enumerate(st.factors):
            prev = st.inverses[k] if st.inverses is not None else None
            new.append(guarded_root_inverse(f / corr, p, cfg.exponent_multiplier, cfg.epsilon,
                                            cfg.solver, cfg.newton_tolerance, prev, self.guard))
        st.inverses = new
        st.last_inverse_step = t

    def _fallback_update(self, st: OracleBlockState, g):  # precond.py:305-313, 355-364
        beta2 = self.cfg.betas[1]
        if st.kind == "adagrad":
            sq = (g * g).astype(st.diag_acc.dtype, copy=False)
            if beta2 == 1.0:
                st.diag_acc += sq
            else:
                st.diag_acc *= beta2
                st.diag_acc += (1.0 - beta2) * sq
        else:
            for k, dvec in enumerate(st.diags):
                other = tuple(a for a in range(g.ndim) if a != k)
                sq = (np.sum(g * g, axis=other) if other else g * g).astype(dvec.dtype, copy=False)
                if beta2 == 1.0:
                    dvec += sq
                else:
                    dvec *= beta2
                    dvec += (1.0 - beta2) * sq
        st.step += 1

    def _fallback_precondition(self, st: OracleBlockState, g, t):  # precond.py:315-320, 366-396
        cfg = self.cfg
        beta2 = cfg.betas[1]
        corr = 1.0 - beta2 ** (t + 1) if (cfg.use_bias_correction and beta2 < 1.0) else 1.0
        if st.kind == "adagrad":
            acc = np.asarray(st.diag_acc, dtype=np.float64) / corr
            return g / (np.sqrt(acc) + cfg.grafting_epsilon)
        out = np.asarray(g, dtype=np.float64)
        expo = -cfg.exponent_multiplier / self.root_p(len(st.shape))
        for k, dvec in enumerate(st.diags):
            scale = (np.asarray(dvec, dtype=np.float64) / corr + cfg.epsilon) ** expo
            shp = [1] * len(st.shape)
            shp[k] = st.shape[k]
            out = out * scale.reshape(shp)
        return out

    # -- the step

    def block_direction(self, i: int, b: int, g, t: int) -> np.ndarray:
        """optim.py:278-344, in the same order of operations."""
        cfg = self.cfg
        st = self.states[i][b]
        if st is None:
            raise ValueError("block not owned")
        w = self.merged(i)[tuple(slice(lo, hi) for lo, hi in self.plans[i][2][b])]
        g = np.asarray(g, dtype=np.float64)
        if cfg.weight_decay > 0.0 and not cfg.use_decoupled_weight_decay:
            g = g + cfg.weight_decay * w
        if st.kind == "shampoo":
            self._factor_update(st, g)
        elif st.kind in ("adagrad", "diagonal"):
            self._fallback_update(st, g)
        self._graft_update(st, g)
        if st.kind == "shampoo":
            self._maybe_refresh(st, t)
        beta1 = cfg.betas[0]
        if beta1 > 0.0:
            st.filtered *= beta1
            st.filtered += (1.0 - beta1) * g
            g_eff = (st.filtered / (1.0 - beta1 ** (t + 1)) if cfg.use_bias_correction
                     else st.filtered.copy())
        else:
            g_eff = g
        p_graft = self._graft_direction(st, g_eff)
        p = p_graft
        if t >= cfg.start_preconditioning_step and st.kind != "graft_only":
            if st.kind == "shampoo" and st.inverses is not None:
                d = np.asarray(g_eff, dtype=np.float64)
                for k, inv in enumerate(st.inverses):
                    d = mode_apply(np.asarray(inv, dtype=np.float64), d, k)
                p = self._rescale(d, p_graft)
            elif st.kind in ("adagrad", "diagonal"):
                p = self._rescale(self._fallback_precondition(st, g_eff, t), p_graft)
        if cfg.weight_decay > 0.0 and cfg.use_decoupled_weight_decay:
            p = p + cfg.weight_decay * w
        if cfg.momentum > 0.0:
            st.momentum *= cfg.momentum
            st.momentum += p
            p = cfg.momentum * st.momentum + p if cfg.use_nesterov else st.momentum
        return p

    @staticmethod
    def _rescale(p_sh, p_graft):
        """p = -rescale_to_graft(p_sh, p_graft) (grafting.py:95-110, optim.py:324)."""
        n_sh = float(np.linalg.norm(p_sh))
        if n_sh == 0.0:
            return np.asarray(p_graft, dtype=np.float64)
        return (float(np.linalg.norm(p_graft)) / n_sh) * p_sh

    def apply_directions(self, directions: dict, t: int) -> None:  # optim.py:346-354
        lr = lr_at(self.cfg, t)
        for (i, b), p in directions.items():
            sl = tuple(slice(lo, hi) for lo, hi in self.plans[i][2][b])
            self.merged(i)[sl] -= lr * p

    def step(self, grads) -> dict:
        """optim.py:356-383. Returns the per-block directions (for parity checks)."""
        if len(grads) != len(self.params):
            raise ValueError("gradient count mismatch")
        for g in grads:
            if not np.all(np.isfinite(g)):
                raise FloatingPointError("non-finite gradient")
        t = self.t
        dirs = {}
        for i, g in enumerate(grads):
            if tuple(np.shape(g)) != self.params[i].shape:
                raise ValueError("gradient shape mismatch")
            gm = np.asarray(g, dtype=np.float64).reshape(self.plans[i][0])
            for b, r in enumerate(self.plans[i][2]):
                if self.states[i][b] is None:
                    continue
                dirs[(i, b)] = self.block_direction(i, b, gm[tuple(slice(lo, hi) for lo, hi in r)], t)
        self.apply_directions(dirs, t)
        self.t += 1
        return dirs


# ---------------------------------------------------------------- sharded simulation


def distributed_step(workers: list[OracleShampoo], plan: OracleAssignment, blocks, grads):
    """dist.py:332-369: owners compute, rank-ordered regions are concatenated, all apply.

    ``workers[r]`` must have been built with owned = plan.owned(r).  Returns the
    flat gather buffer of group 0 (float64 scalars) for layout checks.
    """
    for g in grads:
        if not np.all(np.isfinite(g)):
            raise FloatingPointError("non-finite gradient")
    G = plan.group_size
    first = None
    for g0 in range(0, plan.world_size, G):
        buf = np.zeros(plan.buffer_scalars)
        group = workers[g0:g0 + G]
        for w in group:
            t = w.t
            for gid in plan.owned(workers.index(w)):
                blk = blocks[gid]
                gm = np.asarray(grads[blk.param_index], dtype=np.float64).reshape(
                    w.plans[blk.param_index][0])
                d = w.block_direction(blk.param_index, blk.block_index, gm[blk.slices], t)
                buf[plan.offsets[gid]:plan.offsets[gid] + blk.var_count] = d.reshape(-1)
        for w in group:
            dirs = {(blk.param_index, blk.block_index):
                    buf[plan.offsets[blk.block_id]:plan.offsets[blk.block_id] + blk.var_count]
                    .reshape(blk.shape) for blk in blocks}
            w.apply_directions(dirs, w.t)
            w.t += 1
        if first is None:
            first = buf
    return first
