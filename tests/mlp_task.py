"""The reference trainer's synthetic MLP task, restated for the acceptance tests (test infrastructure).

Data, split, initialisation and batch sampling follow minishampoo/train.py (pinned to the real
reference by tests/golden/acceptance11.json through test_acceptance.py::test_mlp_task_pinned):

  stream_rng            train.py:58-60    np.random.default_rng([seed, *lanes])
  make_synthetic_classes train.py:229-251 ill-conditioned Gaussian clusters, 10% label noise
  prepare_bundle        train.py:272-298  seeded split, per-feature standardisation
  Mlp.initialize        train.py:87-94    uniform(+-sqrt(6 / (fan_in + fan_out))), (fan_out, fan_in)
  batch_at              train.py:301-308  indices = stream_rng(seed, 3, step).integers(0, n, B)
  forward / loss        train.py:118-196  bias-free ReLU MLP, mean softmax cross-entropy
"""

from __future__ import annotations

import math

import numpy as np

LANE_INIT, LANE_DATA, LANE_SPLIT, LANE_BATCH = 0, 1, 2, 3


def stream_rng(seed: int, *lanes: int) -> np.random.Generator:
    return np.random.default_rng([int(seed), *[int(x) for x in lanes]])


def make_synthetic_classes(seed: int, classes: int, dim: int, count: int):
    rng = stream_rng(seed, LANE_DATA)
    means = rng.normal(0.0, 1.0, size=(classes, dim))
    scales = rng.uniform(0.5, 1.5, size=(classes, dim))
    labels = rng.integers(0, classes, size=count)
    clusters = means[labels] + rng.standard_normal((count, dim)) * scales[labels]
    left, _ = np.linalg.qr(rng.standard_normal((dim, dim)))
    right, _ = np.linalg.qr(rng.standard_normal((dim, dim)))
    mixing = (left * 10.0 ** np.linspace(-1.5, 1.5, dim)) @ right.T
    flip = rng.random(count) < 0.1
    labels = np.where(flip, rng.integers(0, classes, size=count), labels)
    return clusters @ mixing.T, labels


def prepare_bundle(features, labels, seed: int, val_fraction: float = 0.2):
    count = len(features)
    perm = stream_rng(seed, LANE_SPLIT).permutation(count)
    n_val = int(round(count * val_fraction))
    val_idx, train_idx = perm[:n_val], perm[n_val:]
    train_x, val_x = features[train_idx], features[val_idx]
    train_y, val_y = labels[train_idx], labels[val_idx]
    mean, std = train_x.mean(axis=0), train_x.std(axis=0)
    std = np.where(std == 0.0, 1.0, std)
    return (train_x - mean) / std, train_y, (val_x - mean) / std, val_y


def init_weights(widths, seed: int):
    rng = stream_rng(seed, LANE_INIT)
    out = []
    for fan_in, fan_out in zip(widths, widths[1:]):
        s = math.sqrt(6.0 / (fan_in + fan_out))
        out.append(rng.uniform(-s, s, size=(fan_out, fan_in)))
    return out


def batch_indices(seed: int, step: int, n_train: int, batch_size: int) -> np.ndarray:
    return stream_rng(seed, LANE_BATCH, step).integers(0, n_train, size=batch_size)


def acceptance11_task(seed: int = 0):
    """test_acceptance.py:288-293: 10 classes, 32 features, 8192 samples, widths [32, 64, 10]."""
    features, labels = make_synthetic_classes(seed, classes=10, dim=32, count=8192)
    train_x, train_y, val_x, val_y = prepare_bundle(features, labels, seed)
    return train_x, train_y, init_weights([32, 64, 10], seed)
