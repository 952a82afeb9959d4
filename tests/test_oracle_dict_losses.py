"""Pins the CPU oracle's decoder and losses against the reference's own suites
(proj/tests/test_dictionary.cpp, proj/tests/test_losses.cpp)."""
import math

import numpy as np
import pytest

import oracle
from tests.helpers import grad_check


def random_state(k, ds, df, rng):  # test_dictionary.cpp:15-24
    atoms = rng.standard_normal((k, df))
    proj = rng.standard_normal((ds, df)) * 0.5
    return oracle.Dictionary(atoms, atoms.copy(), proj, 1.0)


def attention_reconstruct(q, proj, atoms, tau):  # oracles.hpp:96-119 (triple loop)
    n, ds = q.shape
    k, df = atoms.shape
    out = np.zeros((n, df))
    for r in range(n):
        logits = np.array([sum(q[r, a] * proj[a, b] * atoms[j, b] for a in range(ds) for b in range(df))
                           for j in range(k)]) / tau
        m = logits.max()
        z = np.exp(logits - m).sum()
        for j in range(k):
            out[r] += math.exp(logits[j] - m) / z * atoms[j]
    return out


def test_single_atom_returns_atom():  # test_dictionary.cpp:35-41
    rng = np.random.default_rng(1)
    st = random_state(1, 3, 5, rng)
    f = oracle.reconstruct(rng.standard_normal((4, 3)), st.atoms, st.proj, 1.0)
    assert np.abs(f - st.atoms[0]).max() < 1e-12


def test_saturated_margin_selects_atom():  # test_dictionary.cpp:43-52
    atoms = np.eye(6)
    q = np.zeros((1, 6))
    q[0, 2] = 50.0
    f = oracle.reconstruct(q, atoms, np.eye(6), 1.0)
    assert np.abs(f[0] - atoms[2]).max() < 1e-9


def test_reconstruct_triple_loop():  # test_dictionary.cpp:54-61
    rng = np.random.default_rng(3)
    st = random_state(6, 3, 5, rng)
    q = rng.standard_normal((4, 3))
    f = oracle.reconstruct(q, st.atoms, st.proj, 1.0)
    assert np.abs(f - attention_reconstruct(q, st.proj, st.atoms, 1.0)).max() < 1e-6


def test_rows_sum_to_one_and_hull():  # test_dictionary.cpp:63-78
    rng = np.random.default_rng(4)
    for _ in range(20):
        st = random_state(7, 4, 6, rng)
        q = rng.standard_normal((9, 4)) * 2
        f, att = oracle.reconstruct(q, st.atoms, st.proj, 1.0, want_attention=True)
        np.testing.assert_allclose(att.sum(1), 1.0, rtol=1e-6)
        assert np.all(f >= st.atoms.min(0) - 1e-9) and np.all(f <= st.atoms.max(0) + 1e-9)


def test_backward_degeneracies():  # test_dictionary.cpp:87-106
    rng = np.random.default_rng(6)
    st = random_state(1, 3, 5, rng)
    q = rng.standard_normal((4, 3))
    _, att = oracle.reconstruct(q, st.atoms, st.proj, 1.0, want_attention=True)
    g = oracle.reconstruct_backward(q, att, st.atoms, st.proj, 1.0, np.zeros((4, 5)))
    assert all(np.abs(g[k]).max() == 0 for k in ("d_queries", "d_proj", "d_atoms"))
    g = oracle.reconstruct_backward(q, att, st.atoms, st.proj, 1.0, rng.standard_normal((4, 5)))
    assert np.abs(g["d_queries"]).max() < 1e-12 and np.abs(g["d_proj"]).max() < 1e-12
    assert np.abs(g["d_atoms"]).max() > 0


def test_backward_fd():  # test_dictionary.cpp:108-127
    rng = np.random.default_rng(7)
    st = random_state(6, 3, 5, rng)
    q = rng.standard_normal((4, 3))
    up = rng.standard_normal((4, 5))
    _, att = oracle.reconstruct(q, st.atoms, st.proj, 1.0, want_attention=True)
    g = oracle.reconstruct_backward(q, att, st.atoms, st.proj, 1.0, up)
    loss = lambda: float((oracle.reconstruct(q, st.atoms, st.proj, 1.0) * up).sum())  # noqa: E731
    assert grad_check(loss, q, g["d_queries"]) < 1e-4
    assert grad_check(loss, st.proj, g["d_proj"]) < 1e-4
    assert grad_check(loss, st.atoms, g["d_atoms"]) < 1e-4


def test_checksum_detects_state_change():  # test_dictionary.cpp:129-138 (stale-cache pin)
    rng = np.random.default_rng(8)
    st = random_state(5, 3, 4, rng)
    c0 = oracle.dictionary_checksum(st.atoms, st.proj)
    st.atoms[0, 0] += 1.0
    assert oracle.dictionary_checksum(st.atoms, st.proj) != c0


def test_trust_region_hinge():  # test_dictionary.cpp:140-154
    rng = np.random.default_rng(9)
    anchor = rng.standard_normal((5, 4))
    atoms = anchor.copy()
    p, g = oracle.trust_region_penalty(atoms, anchor, 0.1, want_grad=True)
    assert p == 0.0 and np.abs(g).max() == 0
    atoms[2, 0] += 0.15
    p, g = oracle.trust_region_penalty(atoms, anchor, 0.1, want_grad=True)
    assert p == pytest.approx(0.05, rel=1e-9)
    assert g[2, 0] == pytest.approx(1.0, rel=1e-9)
    assert np.abs(g[0]).max() == 0


def test_trust_region_scalar_oracle_and_fd():  # test_dictionary.cpp:156-181
    rng = np.random.default_rng(10)
    anchor = rng.standard_normal((6, 5))
    atoms = anchor + rng.standard_normal((6, 5)) * 0.2
    expect = sum(max(0.0, np.linalg.norm(anchor[j] - atoms[j]) - 0.3) for j in range(6))
    p, g = oracle.trust_region_penalty(atoms, anchor, 0.3, want_grad=True)
    assert p == pytest.approx(expect, rel=1e-12)
    for j in range(6):
        if abs(np.linalg.norm(atoms[j] - anchor[j]) - 0.3) < 1e-3:
            continue
        row = atoms[j]
        loss = lambda: float(oracle.trust_region_penalty(atoms, anchor, 0.3))  # noqa: E731
        assert grad_check(loss, row, g[j]) < 1e-5


def test_trust_region_lipschitz():  # test_dictionary.cpp:183-196
    rng = np.random.default_rng(11)
    anchor = rng.standard_normal((4, 6))
    for _ in range(200):
        a = anchor + rng.standard_normal((4, 6)) * 0.3
        b = a.copy()
        j = rng.integers(4)
        step = rng.standard_normal(6) * 0.05
        b[j] += step
        pa = oracle.trust_region_penalty(a, anchor, 0.2)
        pb = oracle.trust_region_penalty(b, anchor, 0.2)
        assert abs(pb - pa) <= np.linalg.norm(step) + 1e-12


# ---------------------------------------------------------------------------- losses
def ssim_reference(a, b):  # oracles.hpp:123-194 (direct 2-D convolution)
    win, rad = 11, 5
    c1, c2 = 1e-4, 9e-4
    ii = np.arange(win) - rad
    kern = np.exp(-(ii[:, None] ** 2 + ii[None, :] ** 2) / (2 * 1.5 * 1.5))
    kern /= kern.sum()
    h, w = a.shape[:2]
    a3 = a.reshape(h, w, -1)
    b3 = b.reshape(h, w, -1)
    if h < win or w < win:
        tot = 0
        for c in range(a3.shape[2]):
            x, y = a3[..., c], b3[..., c]
            mx, my = x.mean(), y.mean()
            vx, vy, cov = ((x - mx) ** 2).mean(), ((y - my) ** 2).mean(), ((x - mx) * (y - my)).mean()
            tot += (2 * mx * my + c1) * (2 * cov + c2) / ((mx * mx + my * my + c1) * (vx + vy + c2))
        return tot / a3.shape[2]

    def refl(i, n):
        return np.where(i < 0, -i, np.where(i >= n, 2 * n - 2 - i, i))

    tot = 0
    ys, xs = np.arange(h), np.arange(w)
    for c in range(a3.shape[2]):
        x, y = a3[..., c], b3[..., c]
        mx = np.zeros((h, w)); my = np.zeros((h, w)); ex2 = np.zeros((h, w)); ey2 = np.zeros((h, w))
        exy = np.zeros((h, w))
        for i in range(-rad, rad + 1):
            for j in range(-rad, rad + 1):
                yy = refl(ys + i, h)[:, None]
                xx = refl(xs + j, w)[None, :]
                kw = kern[i + rad, j + rad]
                av, bv = x[yy, xx], y[yy, xx]
                mx += kw * av; my += kw * bv; ex2 += kw * av * av; ey2 += kw * bv * bv; exy += kw * av * bv
        sx2, sy2, sxy = ex2 - mx * mx, ey2 - my * my, exy - mx * my
        tot += ((2 * mx * my + c1) * (2 * sxy + c2) / ((mx * mx + my * my + c1) * (sx2 + sy2 + c2))).sum()
    return tot / (h * w * a3.shape[2])


def test_ssim_identical_is_one():  # test_losses.cpp:23-27
    a = np.random.default_rng(1).random((24, 32, 3))
    assert oracle.ssim(a, a) == pytest.approx(1.0, rel=1e-9)


def test_ssim_inverted_checkerboard_negative():  # test_losses.cpp:29-36
    a = np.zeros((24, 32, 1))
    for y in range(24):
        for x in range(32):
            a[y, x] = 1.0 if (x // 4 + y // 4) % 2 else 0.0
    assert oracle.ssim(a, 1.0 - a) < 0.0


def test_ssim_direct_convolution_oracle():  # test_losses.cpp:38-46
    rng = np.random.default_rng(2)
    for _ in range(5):
        a, b = rng.random((20, 26, 3)), rng.random((20, 26, 3))
        assert oracle.ssim(a, b) == pytest.approx(ssim_reference(a, b), rel=1e-6)


def test_ssim_small_image_fallback():  # test_losses.cpp:48-55
    rng = np.random.default_rng(3)
    a, b = rng.random((6, 7, 1)), rng.random((6, 7, 1))
    assert oracle.ssim(a, b) == pytest.approx(ssim_reference(a, b), rel=1e-9)
    assert oracle.ssim(a, a) == pytest.approx(1.0, rel=1e-9)


def test_ssim_gradient_fd():  # test_losses.cpp:57-76
    rng = np.random.default_rng(4)
    a, b = rng.random((16, 18, 1)), rng.random((16, 18, 1))
    _, da = oracle.ssim(a, b, want_grad=True)
    assert grad_check(lambda: float(oracle.ssim(a, b)), a, da, 1e-5, 60) < 1e-4
    sa, sb = rng.random((6, 6, 2)), rng.random((6, 6, 2))
    _, dsa = oracle.ssim(sa, sb, want_grad=True)
    assert grad_check(lambda: float(oracle.ssim(sa, sb)), sa, dsa, 1e-5) < 1e-4


def test_rgb_loss_exact_and_offset():  # test_losses.cpp:78-96
    img = np.random.default_rng(5).random((24, 32, 3))
    assert oracle.rgb_loss(img, img, 0.2, 0.8, False)["value"] == pytest.approx(0.0, abs=1e-12)
    flat = np.full((24, 32, 3), 0.4)
    r = oracle.rgb_loss(flat + 0.1, flat, 0.2, 0.8, False)
    assert r["l1"] == pytest.approx(0.1, rel=1e-9)
    lum = (2 * 0.5 * 0.4 + 1e-4) / (0.25 + 0.16 + 1e-4)
    assert r["ssim_loss"] == pytest.approx((1 - lum) / 2, rel=1e-6)


def test_rgb_loss_fd():  # test_losses.cpp:98-107
    rng = np.random.default_rng(6)
    a, b = rng.random((16, 16, 3)), rng.random((16, 16, 3))
    r = oracle.rgb_loss(a, b, 0.2, 0.8, True)
    assert grad_check(lambda: float(oracle.rgb_loss(a, b, 0.2, 0.8, False)["value"]), a, r["grad"],
                      1e-5, 60) < 1e-4


def test_depth_loss_masks():  # test_losses.cpp:109-137
    alpha = np.ones((4, 4))
    z = np.full((4, 4), 2.0)
    assert oracle.depth_loss(z.copy(), z, alpha, False)["value"] == 0.0
    assert oracle.depth_loss(z + 0.05, z, alpha, False)["value"] == pytest.approx(0.05, rel=1e-12)
    z2 = z.copy()
    z2[:, :2] = 0.0
    zr2 = z2 + np.where(np.arange(4)[None, :] >= 2, 0.1, 5.0)
    d = oracle.depth_loss(zr2, z2, alpha, True)
    assert d["value"] == pytest.approx(0.1, rel=1e-12)
    assert d["grad"][0, 0] == 0.0
    assert d["grad"][0, 2] == pytest.approx(1 / 8, rel=1e-12)
    none = oracle.depth_loss(z + 0.05, z, np.zeros((4, 4)), False)
    assert none["flagged"] and none["value"] == 0.0


def test_feature_loss_cases_and_fd():  # test_losses.cpp:139-178
    rng = np.random.default_rng(7)
    f = rng.standard_normal((5, 6))
    atoms = rng.standard_normal((3, 6))
    anchor = atoms.copy()
    fl = oracle.feature_loss(f, f, atoms, anchor, 0.1, 0.5, 0.5, 0.2, False)
    assert fl["value"] == pytest.approx(0.0, abs=1e-12)
    fl = oracle.feature_loss(2 * f, f, atoms, anchor, 0.1, 0.5, 0.5, 0.2, False)
    assert fl["cos_term"] == pytest.approx(0.0, abs=1e-9)
    assert fl["l2_term"] == pytest.approx((f ** 2).sum(1).mean(), rel=1e-9)
    rec = rng.standard_normal((5, 6))
    fl = oracle.feature_loss(rec, f, atoms, anchor, 0.1, 0.5, 0.5, 0.2, True)
    cs = np.mean([1 - rec[r] @ f[r] / (np.linalg.norm(rec[r]) * np.linalg.norm(f[r])) for r in range(5)])
    assert fl["cos_term"] == pytest.approx(cs, rel=1e-9)
    assert fl["l2_term"] == pytest.approx(((rec - f) ** 2).sum(1).mean(), rel=1e-9)
    loss = lambda: float(oracle.feature_loss(rec, f, atoms, anchor, 0.1, 0.5, 0.5, 0.2, False)["value"])  # noqa
    assert grad_check(loss, rec, fl["d_reconstructed"], 1e-5) < 1e-4


def test_feature_loss_zero_norm_flag():  # test_losses.cpp:180-187
    fl = oracle.feature_loss(np.zeros((2, 3)), np.ones((2, 3)), np.ones((2, 3)), np.ones((2, 3)), 0.1, 1, 1,
                             1, False)
    assert fl["zero_norm_flagged"] and np.isfinite(fl["value"])
