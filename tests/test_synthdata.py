"""Seeded input generators (synthdata/): known-answer PRNG vector, distribution checks, SHA fixtures."""
import json
import os

import numpy as np
import pytest

import synthdata as sd

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_vector():
    # the published splitmix64 test vector for seed 1234567 (Vigna's splitmix64.c)
    assert [int(v) for v in sd.splitmix64(1234567, 0, 5)] == [
        6457827717110365317, 3203168211198807973, 9817491932198370423,
        4593380528125082431, 16408922859458223821]


def test_stream_offsets_are_consistent():
    a = sd.splitmix64(42, 0, 100)
    b = sd.splitmix64(42, 37, 20)
    np.testing.assert_array_equal(a[37:57], b)


def test_uniform_moments():
    u = sd.uniform01(3, 0, 1 << 20)
    assert 0.0 <= u.min() and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 2e-3
    assert abs(u.var() - 1 / 12) < 1e-3
    # 24-bit values are exact in fp32
    np.testing.assert_array_equal(u.astype(np.float32).astype(np.float64), u)


def test_config0_dataset():
    d = sd.make_dataset(sd.WORKLOADS["config0"])
    assert d.x_train.shape == (1000, 841) and d.x_test.shape == (200, 841)
    assert d.x_train.dtype == np.float32 and d.y_train.dtype == np.int32
    assert d.x_train.min() >= -1 and d.x_train.max() <= 1
    assert abs(d.x_train.mean()) < 5e-3 and abs(d.x_train.var() - 1 / 3) < 5e-3
    assert set(np.unique(d.y_train)) <= set(range(10))


def test_prototype_dataset_structure():
    d = sd.prototype_dataset(1, 3000, 500)
    assert d.x_train.min() >= -1 and d.x_train.max() <= 1
    counts = np.bincount(d.y_train, minlength=10)
    assert counts.min() > 200  # labels uniform over 10 classes
    # samples of one class scatter around one prototype: class means are far apart
    means = np.stack([d.x_train[d.y_train == c].mean(0) for c in range(10)])
    dist = np.linalg.norm(means[:, None] - means[None], axis=-1)
    assert dist[~np.eye(10, dtype=bool)].min() > 5.0
    # test set continues the stream: it equals samples n_train.. of the same stream
    xs, ys = sd.prototype_samples(1, 3000, 500)
    np.testing.assert_array_equal(xs, d.x_test)
    np.testing.assert_array_equal(ys, d.y_test)


def test_init_bounds_and_order():
    blocks = [(16, 80, 5), (845, 8450, 10)]
    p = sd.init_params(0, blocks)
    assert p.dtype == np.float32 and p.shape == (8545,)
    assert np.abs(p[:85]).max() <= 0.25 and np.abs(p[:85]).max() > 0.2
    assert np.abs(p[85:]).max() <= 1 / np.sqrt(845) + 1e-7
    # drawn from seed data_seed ^ 0x5EED, consecutive draws
    u = sd.uniform01(0 ^ 0x5EED, 0, 85)
    np.testing.assert_allclose(p[:85], ((2 * u - 1) * 0.25).astype(np.float32))


def test_dataset_sha256_fixture():
    ref = json.load(open(os.path.join(GOLD, "data_sha256.json")))
    assert sd.make_dataset(sd.WORKLOADS["config0"]).sha256() == ref["config0"]
    assert sd.make_dataset(sd.WORKLOADS["config1"], 2000, 200).sha256() == ref["config1_prefix2000_test200"]
