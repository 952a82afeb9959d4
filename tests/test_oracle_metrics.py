"""Oracle pin for the evaluation metrics: metric_cos, metric_miou,
metric_psnr (proj/src/metrics.cpp:8-89) and query_map scores (proj/src/evaluate.cpp:74-88) against
the reference's own cases (proj/tests/test_io.cpp:128-225)."""
import math

import numpy as np
import pytest

import oracle


def test_metric_cos_examples():  # test_io.cpp:128-143
    f = np.array([[1, 0, 0, 0], [0, 2, 0, 0], [0.3, 0.3, 0, 0]], np.float32)
    # the reference checks 0 within 1e-9; with float row norms (Eigen's norm() on a float row, as
    # restated) the (0.3, 0.3) row leaves sqrtf rounding of ~1.8e-8, i.e. 5.9e-9 on the mean
    assert oracle.metric_cos(f, f)[0] == pytest.approx(0.0, abs=1e-8)
    assert oracle.metric_cos(f, -f)[0] == pytest.approx(2.0, rel=1e-6)
    assert oracle.metric_cos(np.array([[1, 0]], np.float32), np.array([[0, 1]], np.float32))[0] == pytest.approx(1.0)
    _, flagged = oracle.metric_cos(np.zeros((1, 2), np.float32), np.array([[0, 1]], np.float32))
    assert flagged


def test_metric_miou_exact_constant_bruteforce():  # test_io.cpp:145-199
    protos = np.eye(3, dtype=np.float32)
    emb = np.array([[1, 0, 0], [0, 1, 0], [0, 1, 0], [0, 0, 1]], np.float32)
    assert oracle.metric_miou(emb, [0, 1, 1, 2], protos)[0] == pytest.approx(1.0)
    const_a = np.tile(np.array([[1, 0, 0]], np.float32), (4, 1))
    m, inter, uni = oracle.metric_miou(const_a, [0, 0, 1, 1], protos)
    assert m == pytest.approx(0.25)
    assert inter[0] / uni[0] == pytest.approx(0.5) and uni[2] == 0  # class 2 absent: excluded
    g = np.random.default_rng(9)
    re = g.standard_normal((50, 3)).astype(np.float32)
    rl = g.integers(0, 3, 50).astype(np.int32)
    got = oracle.metric_miou(re, rl, protos)[0]
    pred = np.argmax(re @ protos.T, axis=1)
    inter = np.zeros(3)
    uni = np.zeros(3)
    for p, t in zip(pred, rl):
        if p == t:
            inter[p] += 1
            uni[p] += 1
        else:
            uni[p] += 1
            uni[t] += 1
    expect = np.mean([inter[c] / uni[c] for c in range(3) if uni[c]])
    assert got == pytest.approx(expect, rel=1e-12)
    with pytest.raises(ValueError):
        oracle.metric_miou(re, np.full(50, 3, np.int32), protos)
    # unlabeled pixels are skipped
    assert oracle.metric_miou(emb, [-1, -1, -1, -1], protos)[0] == 0.0


def test_metric_psnr_examples():  # test_io.cpp:201-225
    a = (np.arange(8 * 8 * 3) % 17 / np.float32(17.0)).astype(np.float32)
    db, exact = oracle.metric_psnr(a, a)
    assert exact and db == 100.0
    b = (a + np.float32(0.1)).astype(np.float32)
    db, exact = oracle.metric_psnr(b, a)
    assert not exact and db == pytest.approx(20.0, rel=1e-4)
    c = np.random.default_rng(11).uniform(0, 1, a.shape).astype(np.float32)
    mse = np.mean((c.astype(np.float64) - a.astype(np.float64)) ** 2)
    assert oracle.metric_psnr(c, a)[0] == pytest.approx(10 * math.log10(1 / mse), rel=1e-9)


def test_query_scores_cosines():
    g = np.random.default_rng(3)
    rec = g.standard_normal((20, 8)).astype(np.float32)
    e = g.standard_normal(8).astype(np.float32)
    s = oracle.query_scores(rec, e)
    ref = rec.astype(np.float64) @ e / (np.linalg.norm(rec, axis=1) * np.linalg.norm(e))
    assert np.allclose(s, ref, rtol=1e-5, atol=1e-6)
    assert oracle.query_scores(np.zeros((1, 8), np.float32), e)[0] == 0.0
