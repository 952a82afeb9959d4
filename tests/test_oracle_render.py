"""Pins the CPU oracle's renderer against the reference's own render tests
(proj/tests/test_render.cpp). Each test cites the reference case it restates."""
import math

import numpy as np
import pytest

import oracle
from tests.helpers import grad_check, random_map, small_intrinsics

A_MAX = 0.999


def example_intr():
    # test_render.cpp:27-35
    return oracle.make_intr(100, 100, 32, 24, 64, 48)


def simple(pos, scale, logit=0.0, qd=4, dtype=np.float64):
    m = oracle.GaussianMap(np.array([pos], dtype), np.array([[1, 0, 0, 0]], dtype),
                           np.array([[0.5, 0.5, 0.5]], dtype), np.full((1, 3), math.log(scale), dtype),
                           np.array([logit], dtype), np.zeros((1, qd), dtype))
    return m


def test_project_principal_point():  # test_render.cpp:38-45
    r = oracle.project_gaussian((0, 0, 1), (1, 0, 0, 0), [math.log(0.05)] * 3, 0.0, (1, 0, 0, 0),
                                (0, 0, 0), example_intr())
    assert r is not None
    mean, cov, depth = r
    assert mean[0] == pytest.approx(32.0, rel=1e-9)
    assert mean[1] == pytest.approx(24.0, rel=1e-9)
    assert depth == pytest.approx(1.0)


def test_project_on_axis_covariance():  # test_render.cpp:47-60
    s, z, fx = 0.08, 2.0, 100
    # positions/log-scales pass through float, as GaussianPrimitive stores float
    r = oracle.project_gaussian((0, 0, np.float32(z)), (1, 0, 0, 0), [float(np.float32(math.log(s)))] * 3,
                                0.0, (1, 0, 0, 0), (0, 0, 0), example_intr())
    mean, cov, depth = r
    expect = (fx * s / z) ** 2 + 0.3
    assert cov[0, 0] == pytest.approx(expect, rel=1e-6)
    assert cov[1, 1] == pytest.approx(expect, rel=1e-6)
    assert abs(cov[0, 1]) < 1e-9


def test_project_culled():  # test_render.cpp:62-68
    intr = example_intr()
    assert oracle.project_gaussian((0, 0, -0.5), (1, 0, 0, 0), [math.log(0.05)] * 3, 0, (1, 0, 0, 0),
                                   (0, 0, 0), intr) is None
    assert oracle.project_gaussian((50, 0, 1.0), (1, 0, 0, 0), [math.log(0.01)] * 3, 0, (1, 0, 0, 0),
                                   (0, 0, 0), intr) is None


def test_single_opaque_gaussian():  # test_render.cpp:70-89
    m = oracle.GaussianMap(np.array([[0, 0, 1.0]]), np.array([[1.0, 0, 0, 0]]), np.array([[0.2, 0.6, 0.9]]),
                           np.full((1, 3), math.log(0.2)), np.array([40.0]), np.array([[1.0, 2, 3, 4]]))
    out = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), example_intr())
    assert out["color"][24, 32, 0] == pytest.approx(0.2 * A_MAX, rel=1e-9)
    assert out["color"][24, 32, 1] == pytest.approx(0.6 * A_MAX, rel=1e-9)
    assert out["query"][24, 32, 3] == pytest.approx(4.0 * A_MAX, rel=1e-9)
    assert out["depth"][24, 32] == pytest.approx(1.0 * A_MAX, rel=1e-9)
    assert out["alpha"][24, 32] == pytest.approx(A_MAX, rel=1e-9)


def test_two_half_opaque_splats():  # test_render.cpp:91-110
    m = oracle.GaussianMap(np.array([[0, 0, 1.0], [0, 0, 2.0]]), np.array([[1.0, 0, 0, 0]] * 2),
                           np.array([[1.0, 0, 0], [0, 1.0, 0]]),
                           np.array([[math.log(0.2)] * 3, [math.log(0.4)] * 3]), np.zeros(2),
                           np.zeros((2, 2)))
    out = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), example_intr())
    assert out["color"][24, 32, 0] == pytest.approx(0.5, rel=1e-9)
    assert out["color"][24, 32, 1] == pytest.approx(0.25, rel=1e-9)
    assert out["alpha"][24, 32] == pytest.approx(0.75, rel=1e-9)


def test_empty_map():  # test_render.cpp:112-118
    m = oracle.GaussianMap(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros((0, 3)),
                           np.zeros(0), np.zeros((0, 3)))
    out = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), example_intr())
    assert out["alpha"][0, 0] == 0.0
    assert out["color"][47, 63, 2] == 0.0


def blend_pixel(splats, m, x, y):
    """Brute-force Eq. 2 restated from oracles.hpp:42-93 (products recomputed from scratch)."""
    hit = [k for k, s in enumerate(splats) if s["x0"] <= x <= s["x1"] and s["y0"] <= y <= s["y1"]]
    hit.sort(key=lambda k: (splats[k]["depth"], splats[k]["source"]))
    a_eff = []
    for k in hit:
        s = splats[k]
        dx, dy = x - s["mean"][0], y - s["mean"][1]
        ci = s["cov_inv"]
        rho = ci[0] * dx * dx + 2 * ci[1] * dx * dy + ci[3] * dy * dy
        a_eff.append(min(A_MAX, s["alpha"] * math.exp(-0.5 * rho)))
    col = np.zeros(3)
    depth = alpha = 0.0
    q = np.zeros(m.ds)
    for i, k in enumerate(hit):
        prod = 1.0
        for j in range(i):
            prod *= 1 - a_eff[j]
        w = a_eff[i] * prod
        src = splats[k]["source"]
        col += w * m.colors[src]
        depth += w * splats[k]["depth"]
        alpha += w
        q += w * m.features[src]
        total = 1.0
        for j in range(i + 1):
            total *= 1 - a_eff[j]
        if total < 1e-4:
            break
    return col, depth, alpha, q


def test_render_matches_brute_force_blend():  # test_render.cpp:120-140
    rng = np.random.default_rng(101)
    intr = small_intrinsics(16, 12, 18.0)
    for trial in range(25):
        m = random_map(12, 3, rng)
        out = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), intr, threads=2)
        for y in range(intr.height):
            for x in range(intr.width):
                col, depth, alpha, q = blend_pixel(out["splats"], m, x, y)
                assert np.abs(out["color"][y, x] - col).max() < 1e-6
                assert abs(out["depth"][y, x] - depth) < 1e-6
                assert abs(out["alpha"][y, x] - alpha) < 1e-6
                assert np.abs(out["query"][y, x] - q).max() < 1e-6
                assert alpha <= 1.0 + 1e-9


def test_render_deterministic_and_order_invariant():  # test_render.cpp:142-168
    rng = np.random.default_rng(55)
    m = random_map(30, 4, rng)
    intr = small_intrinsics(20, 16)
    a = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), intr, threads=1)
    b = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), intr, threads=3)
    assert np.array_equal(a["color"], b["color"]) and np.array_equal(a["query"], b["query"])
    rev = oracle.GaussianMap(*[np.ascontiguousarray(getattr(m, f)[::-1]) for f in oracle.FIELDS])
    c = oracle.render(rev, (1, 0, 0, 0), (0, 0, 0), intr, threads=1)
    np.testing.assert_allclose(a["color"], c["color"], rtol=1e-12, atol=0)


def test_opacity_monotonicity():  # test_render.cpp:170-195
    rng = np.random.default_rng(77)
    m = random_map(10, 2, rng)
    intr = small_intrinsics(16, 12)
    for g in range(3):
        probe = m.copy()
        probe.colors[:] = 0
        probe.colors[g, 0] = 1.0
        before = oracle.render(probe, (1, 0, 0, 0), (0, 0, 0), intr)["color"][..., 0]
        probe.opacity_logits[g] += 0.7
        after = oracle.render(probe, (1, 0, 0, 0), (0, 0, 0), intr)["color"][..., 0]
        mask = before > 1e-12
        assert np.all(after[mask] >= before[mask] - 1e-12)


def test_backward_zero_upstream():  # test_render.cpp:197-210
    rng = np.random.default_rng(31)
    m = random_map(8, 3, rng)
    intr = small_intrinsics()
    out = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), intr)
    h, w = intr.height, intr.width
    g = oracle.render_backward(m, (1, 0, 0, 0), (0, 0, 0), intr, out["splats"], np.zeros((h, w, 3)),
                               np.zeros((h, w)), np.zeros((h, w, 3)))
    assert np.abs(g.positions).max() == 0 and np.abs(g.rotations).max() == 0
    assert np.abs(g.features).max() == 0


class Harness:
    """RenderLossHarness, test_render.cpp:228-256."""

    def __init__(self, intr, rng):
        h, w = intr.height, intr.width
        self.intr = intr
        self.uc = rng.uniform(-1, 1, (h, w, 3))
        self.ud = rng.uniform(-1, 1, (h, w))
        self.uq = rng.uniform(-1, 1, (h, w, 3))

    def loss(self, m):
        out = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), self.intr)
        return float((self.uc * out["color"]).sum() + (self.ud * out["depth"]).sum() +
                     (self.uq * out["query"]).sum())

    def grads(self, m):
        out = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), self.intr)
        return oracle.render_backward(m, (1, 0, 0, 0), (0, 0, 0), self.intr, out["splats"], self.uc, self.ud,
                                      self.uq)


def test_backward_single_gaussian_fd():  # test_render.cpp:269-284
    rng = np.random.default_rng(41)
    m = random_map(1, 3, rng)
    m.opacity_logits[0] = 0.5
    h = Harness(small_intrinsics(), rng)
    g = h.grads(m)
    loss = lambda: h.loss(m)  # noqa: E731
    assert grad_check(loss, m.colors, g.colors) < 1e-4
    assert grad_check(loss, m.positions, g.positions) < 1e-3
    assert grad_check(loss, m.log_scales, g.log_scales) < 1e-3
    assert grad_check(loss, m.rotations, g.rotations) < 1e-3
    assert grad_check(loss, m.opacity_logits, g.opacity_logits) < 1e-4
    assert grad_check(loss, m.features, g.features) < 1e-4


def test_backward_20_gaussian_fd():  # test_render.cpp:286-300
    rng = np.random.default_rng(4242)
    m = random_map(20, 3, rng)
    h = Harness(small_intrinsics(16, 16, 16.0), rng)
    g = h.grads(m)
    loss = lambda: h.loss(m)  # noqa: E731
    assert grad_check(loss, m.positions, g.positions, max_coords=30) < 1e-3
    assert grad_check(loss, m.rotations, g.rotations, max_coords=30) < 1e-3
    assert grad_check(loss, m.colors, g.colors, max_coords=30) < 1e-3
    assert grad_check(loss, m.log_scales, g.log_scales, max_coords=30) < 1e-3
    assert grad_check(loss, m.opacity_logits, g.opacity_logits, max_coords=20) < 1e-3
    assert grad_check(loss, m.features, g.features, max_coords=30) < 1e-3
