"""rgb_loss / depth_loss / feature_loss as standalone C-ABI operators (obj/losses.hpp:12-58),
against the oracle (proj/src/losses.cpp:200-294) on random inputs and on the reference's own
known-answer cases (proj/tests/test_losses.cpp:78-178)."""
import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_12314_b200 import api  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return api.Context(0)


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a, np.float32), device="cuda")


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("h,w,ch", [(48, 64, 3), (7, 9, 3), (120, 160, 1)])
def test_rgb_loss_matches_oracle(ctx, h, w, ch):
    rng = np.random.default_rng(h * w)
    a = rng.random((h, w, ch)).astype(np.float32)
    b = rng.random((h, w, ch)).astype(np.float32)
    got = api.rgb_loss(ctx, dev(a), dev(b), 0.2, 0.8)
    ref = oracle.rgb_loss(a, b, np.float32(0.2), np.float32(0.8))
    for k in ("value", "l1", "ssim_loss"):
        assert got[k] == pytest.approx(float(ref[k]), rel=1e-5, abs=1e-7), k
    assert rel(got["grad"].cpu().numpy(), ref["grad"]) < 1e-4


def test_rgb_loss_known_answer(ctx):
    # test_losses.cpp:78-96: a uniform offset of 0.1 gives l1 = 0.1
    rng = np.random.default_rng(3)
    b = (rng.random((32, 32, 3)) * 0.8).astype(np.float32)
    a = b + np.float32(0.1)
    got = api.rgb_loss(ctx, dev(a), dev(b), 1.0, 0.0)
    assert got["l1"] == pytest.approx(0.1, rel=1e-5)
    g = got["grad"].cpu().numpy()
    assert np.allclose(g, 1.0 / a.size, rtol=1e-6)


def test_depth_loss_matches_oracle_and_flags(ctx):
    rng = np.random.default_rng(11)
    r = (rng.random((40, 50)) * 3).astype(np.float32)
    o = np.where(rng.random((40, 50)) > 0.3, rng.random((40, 50)) * 3, 0.0).astype(np.float32)
    al = rng.random((40, 50)).astype(np.float32)
    got = api.depth_loss(ctx, dev(r), dev(o), dev(al))
    ref = oracle.depth_loss(r, o, al)
    assert got["value"] == pytest.approx(float(ref["value"]), rel=1e-5)
    assert not got["flagged"]
    np.testing.assert_allclose(got["grad"].cpu().numpy(), ref["grad"], rtol=1e-6, atol=0)
    # no valid pixel: flagged, zero value and gradient (test_losses.cpp:128-137)
    got = api.depth_loss(ctx, dev(r), dev(np.zeros_like(o)), dev(al))
    assert got["flagged"] and got["value"] == 0.0 and not got["grad"].cpu().numpy().any()


def test_feature_loss_matches_oracle(ctx):
    rng = np.random.default_rng(5)
    n, df, k = 300, 96, 16
    u = rng.standard_normal((n, df)).astype(np.float32)
    v = rng.standard_normal((n, df)).astype(np.float32)
    anchor = rng.standard_normal((k, df)).astype(np.float32)
    atoms = (anchor + rng.standard_normal((k, df)) * 0.1).astype(np.float32)
    args = (np.float32(0.1), np.float32(0.5), np.float32(0.5), np.float32(0.2))
    got = api.feature_loss(ctx, dev(u), dev(v), dev(atoms), dev(anchor), *args)
    ref = oracle.feature_loss(u, v, atoms, anchor, *args)
    for key in ("value", "cos_term", "l2_term", "trust_term"):
        assert got[key] == pytest.approx(float(ref[key]), rel=1e-5, abs=1e-7), key
    assert rel(got["d_reconstructed"].cpu().numpy(), ref["d_reconstructed"]) < 1e-5
    assert rel(got["d_atoms_trust"].cpu().numpy(), ref["d_atoms_trust"]) < 1e-5
    assert not got["zero_norm_flagged"]


def test_feature_loss_collinear_and_zero_rows(ctx):
    # test_losses.cpp:139-178: identical rows -> cos term 0; a zero row -> flagged
    rng = np.random.default_rng(9)
    u = rng.standard_normal((10, 12)).astype(np.float32)
    atoms = np.zeros((2, 12), np.float32)
    got = api.feature_loss(ctx, dev(u), dev(u * 2.0), dev(atoms), dev(atoms), 0.1, 1.0, 0.0, 0.0)
    assert abs(got["cos_term"]) < 1e-6
    z = u.copy()
    z[3] = 0.0
    got = api.feature_loss(ctx, dev(z), dev(u), dev(atoms), dev(atoms), 0.1, 0.5, 0.5, 0.0)
    ref = oracle.feature_loss(z, u, atoms, atoms, np.float32(0.1), np.float32(0.5), np.float32(0.5), np.float32(0))
    assert got["zero_norm_flagged"] and ref["zero_norm_flagged"]
    assert got["value"] == pytest.approx(float(ref["value"]), rel=1e-5)
