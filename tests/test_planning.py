"""C++ planner through the C ABI: bit-exact against the reference (CPU only, no GPU calls).

Covers precond.py:56-158 (merge/partition/plan) and dist.py:133-243 (enumeration,
greedy assignment, padded layout) -- the reference tests test_precond.py:29-104
and test_dist.py:47-130 restated, plus the model-set fixtures from the real
reference (tests/golden/plans.npz).
"""

from __future__ import annotations

import math
import os
import re

import numpy as np
import pytest

import paper_2309_06497_b200 as P
from oracle import shampoo_oracle as O
from paper_2309_06497_b200 import _native as N
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES
from tests.conftest import ROOT, load_golden


def test_library_exports_every_declared_symbol():
    header = open(f"{ROOT}/include/shampoo_b200.h").read()
    declared = set(re.findall(r"SHAMPOO_API [^;]*?\b(shampoo_\w+)\(", header))
    assert declared == set(N.SIGNATURES), declared ^ set(N.SIGNATURES)
    lib = N.lib()
    for name in declared:
        assert getattr(lib, name) is not None
    assert b"sm_100a" in lib.shampoo_version()


def test_merge_dims_examples():
    assert P.merge_dims((10, 2, 2, 4), 8) == (10, 4, 4)
    assert P.merge_dims((3, 3, 3), 9) == (9, 3)
    assert P.merge_dims((4096, 1), 8) == (4096,)
    assert P.merge_dims((1, 4096, 1, 3), 8) == (4096, 3)
    assert P.merge_dims((), 8) == (1,)
    assert P.merge_dims((4096, 2, 2), 8) == (4096, 4)
    assert P.merge_dims((2, 1024), 8) == (2, 1024)
    with pytest.raises(ValueError):
        P.merge_dims((3, 0), 4)


def test_merge_dims_random_vs_oracle():
    rng = np.random.default_rng(0)
    for _ in range(300):
        shape = tuple(int(d) for d in rng.integers(1, 12, size=int(rng.integers(0, 6))))
        b = int(rng.integers(1, 64))
        assert P.merge_dims(shape, b) == O.merge_dims(shape, b)


def test_plan_parameter_vs_oracle():
    rng = np.random.default_rng(1)
    for _ in range(100):
        shape = tuple(int(d) for d in rng.integers(1, 40, size=int(rng.integers(1, 4))))
        b = int(rng.integers(1, 16))
        for method in P.LargeDimMethod:
            plan = P.plan_parameter(shape, b, method)
            merged, m2, ranges = O.plan_parameter(shape, b, O.LargeDimMethod(method.value))
            assert plan.merged_shape == merged and plan.method.value == m2.value
            assert [s.ranges for s in plan.blocks] == ranges


def test_greedy_worked_example():
    plan = P.greedy_assign([6, 5, 4, 3, 2], world_size=2, group_size=2)
    assert plan.assignments[0] == frozenset({0, 3, 4})
    assert plan.assignments[1] == frozenset({1, 2})
    assert plan.counters == (11, 9)
    assert P.buffer_size(plan) == 176


def test_greedy_edge_cases():
    plan = P.greedy_assign([7], world_size=4, group_size=4)
    assert plan.assignments[0] == frozenset({0})
    assert all(plan.assignments[r] == frozenset() for r in (1, 2, 3))
    assert plan.counters == (7, 0, 0, 0)
    plan = P.greedy_assign([4, 4, 4, 4], 4, 4)
    assert all(len(plan.assignments[r]) == 1 for r in range(4))
    assert P.buffer_size(plan) == 16 * 8
    plan = P.greedy_assign([6, 5, 4, 3, 2], 4, 2)
    assert plan.assignments[0] == plan.assignments[2] and plan.num_groups == 2
    with pytest.raises(P.InvalidGroupSizeError):
        P.greedy_assign([3, 2], world_size=4, group_size=3)
    with pytest.raises(P.InvalidGroupSizeError):
        P.greedy_assign([3], world_size=0, group_size=1)
    with pytest.raises(ValueError):
        P.greedy_assign([3, 0], 2, 2)


def test_greedy_random_vs_oracle_and_layout():
    rng = np.random.default_rng(0)
    for _ in range(200):
        counts = [int(c) for c in rng.integers(1, 400, size=int(rng.integers(1, 12)))]
        group = int(rng.choice([1, 2, 4, 8]))
        world = group * int(rng.choice([1, 2]))
        plan = P.greedy_assign(counts, world, group)
        ref = O.greedy_assign(counts, world, group)
        assert list(plan.counters) == ref.counters
        for i, region in plan.buffer_layout.items():
            assert region.owner_rank == ref.owner[i]
            assert region.scalar_offset == ref.offsets[i]
            start, end = region.byte_offset, region.byte_offset + region.byte_length
            assert region.owner_rank * plan.max_payload_bytes <= start
            assert end <= (region.owner_rank + 1) * plan.max_payload_bytes


PLANS = load_golden("plans.npz")


@pytest.mark.parametrize("key", sorted({k.split("/")[0] for k in PLANS.files}))
def test_model_plans_bit_exact_with_reference(key):
    model, b = key.rsplit("_b", 1)
    shapes = MODEL_SHAPES[model]
    for wk in sorted({k.split("/")[1] for k in PLANS.files if k.startswith(key + "/J")}):
        world, group = (int(v) for v in wk[1:].split("G"))
        plan = P.NativePlan(shapes, int(b), P.LargeDimMethod.BLOCKING, world, group)
        info = plan.blocks_info
        assert [x.param_index for x in info] == PLANS[f"{key}/param_index"].tolist()
        assert [x.block_index for x in info] == PLANS[f"{key}/block_index"].tolist()
        assert [x.var_count for x in info] == PLANS[f"{key}/var_count"].tolist()
        assert [x.owner_rank for x in info] == PLANS[f"{key}/{wk}/owner"].tolist()
        assert [x.gather_offset for x in info] == PLANS[f"{key}/{wk}/offset"].tolist()
        assert list(plan.counters) == PLANS[f"{key}/{wk}/counters"].tolist()
        shp = PLANS[f"{key}/shape"]
        for x, row in zip(info, shp):
            assert tuple(x.hi[k] - x.lo[k] for k in range(x.order)) == tuple(int(v) for v in row if v)


@pytest.mark.parametrize("key", sorted({k.split("/")[0] for k in PLANS.files}))
def test_comm_meter_matches_reference(key):
    """comm_meter (dist.py:394-423) against the reference's own reports for every model plan."""
    model, b = key.rsplit("_b", 1)
    blocks = P.enumerate_blocks(MODEL_SHAPES[model], P.ShampooConfig(max_preconditioner_dim=int(b)))
    for wk in sorted({k.split("/")[1] for k in PLANS.files if k.startswith(key + "/J")}):
        world, group = (int(v) for v in wk[1:].split("G"))
        plan = P.greedy_assign([x.var_count for x in blocks], world, group)
        rep = P.comm_meter(plan, [x.shape for x in blocks], steps=3)
        assert [rep.bytes_gathered_per_step, rep.world_bytes_per_step, rep.total_bytes_gathered] == \
            PLANS[f"{key}/{wk}/comm"].tolist()
        assert list(rep.per_worker_state_scalars) == PLANS[f"{key}/{wk}/state_scalars"].tolist()


def test_resnet50_plan_summary():
    # 161 blocks, orders 1/2/3 = 107/45/9; J=8 buffer 3,194,880 scalars/rank
    plan = P.NativePlan(MODEL_SHAPES["resnet50"], 2048, P.LargeDimMethod.BLOCKING, 8, 8)
    orders = [x.order for x in plan.blocks_info]
    assert len(orders) == 161
    assert (orders.count(1), orders.count(2), orders.count(3)) == (107, 45, 9)
    assert plan.max_payload == 3_194_880
    assert sum(x.var_count for x in plan.blocks_info) == 25_557_032


def test_config_validation_mirrors_reference():
    for kw in [{"betas": (1.0, 0.999)}, {"betas": (0.0, 0.0)}, {"lr": 0.0}, {"momentum": 1.0},
               {"weight_decay": -1.0}, {"precondition_frequency": 0}, {"max_preconditioner_dim": 0},
               {"lr_schedule": "warmup_cosine", "total_steps": 0}, {"lr_schedule": "bogus"},
               {"precision": "half"}, {"grafting_epsilon": 0.0}]:
        with pytest.raises(ValueError):
            P.ShampooConfig(**kw)
    with pytest.raises(ValueError):
        P.ShampooConfig(solver=P.Solver.COUPLED_NEWTON, exponent_multiplier=2.0)


def test_lr_schedule_table():
    cfg = P.ShampooConfig(lr=0.1, lr_schedule="warmup_cosine", warmup_steps=5, total_steps=90)
    for t, v in {0: 0.02, 4: 0.1, 47: 0.050923945247956494, 89: 3.41469928488547e-05}.items():
        assert P.lr_at(cfg, t) == pytest.approx(v, rel=1e-12)
    with pytest.raises(P.OutOfRangeError):
        P.lr_at(cfg, 90)
    assert P.lr_at(P.ShampooConfig(lr=0.3), 10**6) == 0.3


class TestCommMeter:
    """dist.py:394-423, restating test_dist.py:234-274 (TestCommMeter)."""

    def test_matrix_state_accounting(self):
        cfg = P.ShampooConfig(max_preconditioner_dim=8)
        blocks = P.enumerate_blocks([(8, 8)], cfg)
        plan = P.greedy_assign([b.var_count for b in blocks], 1, 1)
        report = P.comm_meter(plan, [b.shape for b in blocks])
        assert report.per_worker_state_scalars == (4 * 64,)
        assert report.per_worker_state_bytes == (4 * 64 * 8,)

    def test_split_matrix_halves_state(self):
        cfg = P.ShampooConfig(max_preconditioner_dim=8)
        blocks = P.enumerate_blocks([(16, 8)], cfg)
        assert len(blocks) == 2
        plan = P.greedy_assign([b.var_count for b in blocks], 2, 2)
        assert P.comm_meter(plan, [b.shape for b in blocks]).per_worker_state_scalars == (4 * 64, 4 * 64)

    def test_cube_state_accounting(self):
        b = 4
        blocks = P.enumerate_blocks([(b, b, b)], P.ShampooConfig(max_preconditioner_dim=b))
        plan = P.greedy_assign([blk.var_count for blk in blocks], 1, 1)
        assert sum(P.comm_meter(plan, [blk.shape for blk in blocks]).per_worker_state_scalars) == 6 * b * b

    def test_gather_volume_scales_with_groups(self):
        plan_one = P.greedy_assign([6, 5, 4, 3], world_size=4, group_size=4)
        plan_two = P.greedy_assign([6, 5, 4, 3], world_size=4, group_size=2)
        shapes = [(6,), (5,), (4,), (3,)]
        one = P.comm_meter(plan_one, shapes, steps=3)
        two = P.comm_meter(plan_two, shapes, steps=3)
        assert one.world_bytes_per_step == P.buffer_size(plan_one)
        assert two.world_bytes_per_step == 2 * P.buffer_size(plan_two)
        assert one.total_bytes_gathered == 3 * one.world_bytes_per_step
        assert set(one.to_json_dict()) == {"steps", "bytes_gathered_per_step", "world_bytes_per_step",
                                           "total_bytes_gathered", "per_worker_state_scalars",
                                           "per_worker_state_bytes"}

    def test_diagonal_fallback_accounting(self):
        plan = P.greedy_assign([12], world_size=1, group_size=1)
        assert P.comm_meter(plan, [(3, 4)], method=P.LargeDimMethod.DIAGONAL).per_worker_state_scalars == (7,)
        assert P.comm_meter(plan, [(3, 4)], method=P.LargeDimMethod.ADAGRAD).per_worker_state_scalars == (12,)
        with pytest.raises(ValueError):
            P.comm_meter(plan, [(3, 4), (2,)])

    def test_resnet50_world8_matches_reference_fixture(self):
        # the J=8 ResNet-50 plan: per-group buffer 204,472,320 B
        blocks = P.enumerate_blocks(MODEL_SHAPES["resnet50"], P.ShampooConfig(max_preconditioner_dim=2048))
        plan = P.greedy_assign([b.var_count for b in blocks], 8, 8)
        report = P.comm_meter(plan, [b.shape for b in blocks], steps=50)
        assert report.bytes_gathered_per_step == 204_472_320
        assert report.total_bytes_gathered == 50 * 204_472_320
        assert sum(report.per_worker_state_scalars) == 2 * 128_111_874


def _plan_case(flags):
    """The reference CLI's flags (RunConfig defaults: input 32, hidden 64, 10 classes) -> inputs."""
    kv = dict(zip(flags[::2], flags[1::2]))
    widths = [32, *[int(w) for w in kv.get("--hidden-widths", "64").split(",")], 10]
    world = int(kv.get("--world-size", 1))
    group = int(kv.get("--num-trainers-per-group", -1))
    cfg = P.ShampooConfig(max_preconditioner_dim=int(kv["--max-preconditioner-dim"]),
                          large_dim_method=P.LargeDimMethod(kv.get("--large-dim-method", "blocking")))
    return P.mlp_param_shapes(widths), cfg, world, (world if group < 0 else group), int(kv.get("--steps", 100))


def test_plan_report_matches_reference_cli():
    """plan_report == the JSON `minishampoo plan` printed (cli.py:168-218), key for key."""
    import json
    cases = json.load(open(os.path.join(ROOT, "tests", "golden", "plan_reports.json")))
    assert len(cases) == 5
    for case in cases:
        shapes, cfg, world, group, steps = _plan_case(case["flags"])
        got = json.loads(json.dumps(P.plan_report(shapes, cfg, world, group, steps), sort_keys=True))
        assert got == case["report"], case["flags"]
