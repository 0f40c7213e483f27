"""Pin the CPU oracle to fixtures produced by the real reference (tests/golden/make_golden.py)."""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import shampoo_oracle as O
from paper_2309_06497_b200.model_shapes import MODEL_SHAPES
from tests.conftest import GOLDEN, load_golden

PLANS = load_golden("plans.npz")
TRAJ = load_golden("trajectories.npz")
RINV = load_golden("rootinv.npz")
META = json.load(open(os.path.join(GOLDEN, "trajectories.json")))

PLAN_KEYS = sorted({k.split("/")[0] for k in PLANS.files})


@pytest.mark.parametrize("key", PLAN_KEYS)
def test_oracle_plan_matches_reference(key):
    model, b = key.rsplit("_b", 1)
    blocks = O.enumerate_blocks(MODEL_SHAPES[model], int(b))
    assert [x.param_index for x in blocks] == PLANS[f"{key}/param_index"].tolist()
    assert [x.block_index for x in blocks] == PLANS[f"{key}/block_index"].tolist()
    assert [x.var_count for x in blocks] == PLANS[f"{key}/var_count"].tolist()
    for wk in sorted({k.split("/")[1] for k in PLANS.files if k.startswith(key + "/J")}):
        world, group = (int(v) for v in wk[1:].split("G"))
        plan = O.greedy_assign([x.var_count for x in blocks], world, group)
        assert plan.owner == PLANS[f"{key}/{wk}/owner"].tolist()
        assert plan.offsets == PLANS[f"{key}/{wk}/offset"].tolist()
        assert plan.counters == PLANS[f"{key}/{wk}/counters"].tolist()


def _oracle_config(name):
    kw = dict(META["configs"][name]["config"])
    enum_fields = {"grafting": O.GraftKind, "solver": O.Solver, "large_dim_method": O.LargeDimMethod}
    for k, e in enum_fields.items():
        if k in kw:
            kw[k] = e(kw[k])
    if "betas" in kw:
        kw["betas"] = tuple(kw["betas"])
    return O.OracleConfig(lr=0.05, **kw)


@pytest.mark.parametrize("name", sorted(META["configs"]))
def test_oracle_trajectory_matches_reference(name):
    cfg = _oracle_config(name)
    shapes = [tuple(s) for s in META["configs"][name]["shapes"]]
    params = [TRAJ[f"{name}/init/{i}"].astype(np.float64) for i in range(len(shapes))]
    opt = O.OracleShampoo(params, cfg)
    for t in range(META["steps"]):
        grads = [TRAJ[f"{name}/grad/{t}/{i}"].astype(np.float64) for i in range(len(shapes))]
        dirs = opt.step(grads)
        for (i, b), d in dirs.items():
            ref = TRAJ[f"{name}/dir/{t}/{i}/{b}"]
            np.testing.assert_allclose(d, ref, rtol=1e-9, atol=1e-12 * max(1.0, np.abs(ref).max()))
        for i in range(len(shapes)):
            np.testing.assert_allclose(opt.params[i], TRAJ[f"{name}/param/{t}/{i}"], rtol=1e-10, atol=1e-12)
    g = META["configs"][name]["guard"]
    assert vars(opt.guard) == g


@pytest.mark.parametrize("case", sorted({k.split("/")[0] for k in RINV.files}))
def test_oracle_root_inverse_matches_reference(case):
    a = RINV[f"{case}/a"]
    for p in (2, 4, 6):
        for eps in (1e-12, 1e-6):
            ref = RINV[f"{case}/eigh/p{p}/e{eps:g}"]
            got = O.root_inverse_eigh(a, p, eps=eps)
            assert np.linalg.norm(got - ref) <= 1e-8 * np.linalg.norm(ref)
    for p in (2, 4):
        key = f"{case}/newton/p{p}"
        if key in RINV.files:
            x, it, _, ok = O.root_inverse_newton(a, p, eps=1e-6)
            assert ok and it == int(RINV[key + "/iters"])
            np.testing.assert_allclose(x, RINV[key], rtol=1e-10, atol=1e-12)
