"""Pin the CPU oracle to the reference's own known-answer tests.

Each test restates a golden vector from /root/reference/pkg/tests (cited) and
checks ``oracle/shampoo_oracle.py`` against it.  CPU only.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import shampoo_oracle as O
from tests.conftest import random_spd, random_symmetric_with_spectrum


def test_merge_dims_examples():  # test_precond.py:29-46
    assert O.merge_dims((10, 2, 2, 4), 8) == (10, 4, 4)
    assert O.merge_dims((3, 3, 3), 9) == (9, 3)
    assert O.merge_dims((5,), 8) == (5,)
    assert O.merge_dims((4096, 1), 8) == (4096,)
    assert O.merge_dims((1, 4096, 1, 3), 8) == (4096, 3)
    assert O.merge_dims((1, 1, 1), 8) == (1,)
    assert O.merge_dims((), 8) == (1,)
    assert O.merge_dims((4096, 2, 2), 8) == (4096, 4)
    assert O.merge_dims((2, 1024), 8) == (2, 1024)


def test_block_partition_example():  # test_precond.py:59-67
    r = O.block_ranges((5, 3), 2)
    assert len(r) == 6
    assert r[0] == ((0, 2), (0, 2)) and r[1] == ((0, 2), (2, 3)) and r[-1] == ((4, 5), (2, 3))


def test_fallback_plan():  # test_precond.py:95-104
    merged, method, ranges = O.plan_parameter((5000, 64), 2048, O.LargeDimMethod.DIAGONAL)
    assert method is O.LargeDimMethod.DIAGONAL and ranges == [((0, 5000), (0, 64))]
    merged, method, ranges = O.plan_parameter((10, 10), 16, O.LargeDimMethod.ADAGRAD)
    assert method is O.LargeDimMethod.BLOCKING


def test_greedy_worked_example():  # test_dist.py:47-52
    plan = O.greedy_assign([6, 5, 4, 3, 2], 2, 2)
    assert plan.owned(0) == [0, 3, 4] and plan.owned(1) == [1, 2]
    assert plan.counters == [11, 9]
    assert plan.buffer_scalars * O.SCALAR_BYTES == 176


def test_greedy_single_block_and_groups():  # test_dist.py:54-72
    plan = O.greedy_assign([7], 4, 4)
    assert plan.owned(0) == [0] and all(plan.owned(r) == [] for r in (1, 2, 3))
    plan = O.greedy_assign([6, 5, 4, 3, 2], 4, 2)
    assert plan.owned(0) == plan.owned(2) and plan.owned(1) == plan.owned(3)
    with pytest.raises(ValueError):
        O.greedy_assign([3, 2], 4, 3)


def test_factor_first_update():  # test_precond.py:142-149
    g = np.array([[1.0, 2.0]])
    assert np.allclose(O.mode_gram(g, 0), [[5.0]])
    assert np.allclose(O.mode_gram(g, 1), [[1.0, 2.0], [2.0, 4.0]])


def test_ema_two_identity_steps():  # test_precond.py:151-157
    cfg = O.OracleConfig(betas=(0.0, 0.999), momentum=0.0, weight_decay=0.0,
                         max_preconditioner_dim=2, start_preconditioning_step=math.inf)
    opt = O.OracleShampoo([np.zeros((2, 2))], cfg)
    opt.step([np.eye(2)])
    opt.step([np.eye(2)])
    st = opt.states[0][0]
    np.testing.assert_allclose(st.factors[0], 0.0019990 * np.eye(2), atol=1e-12)


def test_root_inverse_known_answers():  # test_matfun.py:56-81
    np.testing.assert_allclose(O.root_inverse_eigh(np.diag([16.0, 81.0]), 4),
                               np.diag([0.5, 1 / 3]), atol=1e-14)
    np.testing.assert_allclose(O.root_inverse_eigh(np.diag([16.0]), 4, eta=2.0), [[0.25]], atol=1e-15)
    rng = np.random.default_rng(3)
    a = random_symmetric_with_spectrum(rng, np.array([-1e-8, 2.0]))
    w = np.linalg.eigvalsh(O.root_inverse_eigh(a, 2, eps=1e-12))
    np.testing.assert_allclose(np.sort(w), np.sort(np.array([2 + 1e-8 + 1e-12, 1e-12]) ** -0.5), rtol=1e-6)
    with pytest.raises(O.OracleSolverFailure):
        O.root_inverse_eigh(np.diag([0.0, 1.0]), 2, eps=0.0)


def test_root_inverse_identity_property():  # test_matfun.py:83-91
    rng = np.random.default_rng(11)
    for _ in range(25):
        n = int(rng.integers(1, 17))
        p = int(rng.choice([1, 2, 4]))
        a = random_spd(rng, n, cond=1e6)
        x = O.root_inverse_eigh(a, p)
        assert np.linalg.norm(np.linalg.matrix_power(x, p) @ a - np.eye(n)) <= 1e-6


def test_newton_known_answers():  # test_matfun.py:115-141
    x, it, res, ok = O.root_inverse_newton(np.array([[4.0]]), 2)
    assert ok and abs(x[0, 0] - 0.5) < 1e-6
    x, *_ , ok = O.root_inverse_newton(np.zeros((3, 3)), 2, eps=1e-4)
    np.testing.assert_allclose(x, 100 * np.eye(3), rtol=1e-12)
    rng = np.random.default_rng(21)
    a = random_spd(rng, 8, cond=1e3)
    xn, _, res, ok = O.root_inverse_newton(a, 4)
    xe = O.root_inverse_eigh(a, 4)
    assert ok and np.linalg.norm(xn - xe) <= 1e-6 * np.linalg.norm(xe)


def test_guard_branches():  # test_matfun.py:167-222
    c = O.GuardCounts()
    prev = 7.0 * np.eye(2)
    x = O.guarded_root_inverse(np.full((2, 2), np.nan), 2, 1.0, 1e-12, O.Solver.EIGH, 1e-6, prev, c)
    assert c.fallback_previous == 1 and np.array_equal(x, prev)
    x = O.guarded_root_inverse(np.zeros((2, 2)), 2, 1.0, 0.0, O.Solver.EIGH, 1e-6, None, c)
    assert c.fallback_identity == 1 and np.array_equal(x, np.eye(2))
    x = O.guarded_root_inverse(np.zeros((3, 3)), 2, 1.0, 1e-4, O.Solver.EIGH, 1e-6, None, c)
    np.testing.assert_allclose(x, 100 * np.eye(3))


def test_rescale_worked_example():  # test_grafting.py:66-68 (p = -rescale)
    out = O.OracleShampoo._rescale(np.array([[2.0, 0.0]]), np.array([[0.0, 3.0]]))
    np.testing.assert_allclose(out, [[3.0, 0.0]])
    g = np.array([1.0, -2.0])
    np.testing.assert_array_equal(O.OracleShampoo._rescale(np.zeros(2), g), g)


def test_adam_graft_first_step():  # test_grafting.py:32-40
    cfg = O.OracleConfig(grafting=O.GraftKind.ADAM, grafting_beta2=0.999, momentum=0.0,
                         weight_decay=0.0, start_preconditioning_step=math.inf, lr=1.0)
    opt = O.OracleShampoo([np.zeros(2)], cfg)
    g = np.array([3.0, -4.0])
    d = opt.step([g])[(0, 0)]
    np.testing.assert_allclose(d, g / (np.abs(g) + 1e-8), rtol=1e-12)


def test_nesterov_first_step():  # test_optim.py:271-288
    rng = np.random.default_rng(7)
    w0, g0 = rng.standard_normal(3), rng.standard_normal(3)
    cfg = O.OracleConfig(lr=0.1, betas=(0.0, 1.0), momentum=0.9, use_nesterov=True,
                         weight_decay=0.0, start_preconditioning_step=math.inf)
    opt = O.OracleShampoo([w0.copy()], cfg)
    opt.step([g0])
    np.testing.assert_allclose(opt.params[0], w0 - 0.1 * 1.9 * g0, atol=1e-15)


def test_full_pipeline_closed_form():  # test_optim.py:143-185
    rng = np.random.default_rng(2)
    m, n = 4, 3
    w0 = rng.standard_normal((m, n))
    gs = [rng.standard_normal((m, n)) for _ in range(6)]
    eps, eg, alpha = 1e-10, 1e-8, 0.05
    cfg = O.OracleConfig(lr=alpha, betas=(0.0, 1.0), momentum=0.0, weight_decay=0.0, epsilon=eps,
                         grafting=O.GraftKind.ADAGRAD, grafting_epsilon=eg,
                         precondition_frequency=1, max_preconditioner_dim=4)
    opt = O.OracleShampoo([w0.copy()], cfg)

    def cri(a, p):
        w, q = np.linalg.eigh((a + a.T) / 2)
        w = w - min(w.min(), 0.0) + eps
        return (q * w ** (-1.0 / p)) @ q.T

    w = w0.copy()
    left, right, acc = np.zeros((m, m)), np.zeros((n, n)), np.zeros((m, n))
    for g in gs:
        opt.step([g])
        left += g @ g.T
        right += g.T @ g
        acc += g * g
        psh = cri(left, 4) @ g @ cri(right, 4)
        pg = g / (np.sqrt(acc) + eg)
        w = w - alpha * (np.linalg.norm(pg) / np.linalg.norm(psh)) * psh
        assert np.abs(opt.params[0] - w).max() <= 1e-12


def test_lr_warmup_cosine_table():  # test_optim.py:39-52
    cfg = O.OracleConfig(lr=0.1, lr_schedule="warmup_cosine", warmup_steps=5, total_steps=90)
    table = {0: 0.02, 4: 0.1, 5: 0.1, 47: 0.050923945247956494, 60: 0.027713082211173093,
             89: 3.41469928488547e-05}
    for t, v in table.items():
        assert O.lr_at(cfg, t) == pytest.approx(v, rel=1e-12)


def test_world_size_invariance_small():  # test_dist.py:173-185
    rng = np.random.default_rng(2)
    shapes = [(6, 4), (5,), (3, 3)]
    params = [rng.standard_normal(s) for s in shapes]
    grads = [[rng.standard_normal(s) for s in shapes] for _ in range(6)]
    cfg = O.OracleConfig(lr=0.05, betas=(0.9, 0.999), grafting=O.GraftKind.ADAGRAD,
                         precondition_frequency=1, max_preconditioner_dim=4)
    blocks = O.enumerate_blocks(shapes, 4)
    finals = {}
    for world, group in [(1, 1), (2, 2), (4, 2), (4, 4)]:
        plan = O.greedy_assign([b.var_count for b in blocks], world, group)
        workers = []
        for r in range(world):
            owned = {(blocks[g].param_index, blocks[g].block_index) for g in plan.owned(r)}
            workers.append(O.OracleShampoo([p.copy() for p in params], cfg, owned=owned))
        for g in grads:
            O.distributed_step(workers, plan, blocks, g)
        finals[(world, group)] = workers[0].params
    for key, ps in finals.items():
        for a, b in zip(finals[(1, 1)], ps):
            assert np.abs(a - b).max() <= 1e-12, key
