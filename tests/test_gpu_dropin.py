"""The Eigen-typed drop-in layer (paper_2602_12314_b200/dropin/latmap_dropin.cpp): the reference's
own C++ operator API (proj/include/latmap/**, T = float), linked to the B200 kernels, driven by a
C++ program written against the reference headers (dropin/dropin_check.cpp, built in the
container by __graft_entry__.build()). Every output is replayed through the CPU oracle on the same
inputs; the exception contract (types) is checked too.

Bars as in test_gpu_parity.py: rendered images 1e-4 relative with the 1e-3 floor (+ the query
summation-error scale), splat lists and bboxes exact, gradients 1e-3 with the floor, losses 2e-4."""
import os
import subprocess

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from tests.test_gpu_parity import QUERY_COND, assert_close_floor  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK = os.path.join(ROOT, "paper_2602_12314_b200", "dropin", "_build", "dropin_check")


@pytest.fixture(scope="module")
def out(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(CHECK):
        pytest.fail(f"{CHECK} not built (build() compiles it where /root/reference exists)")
    d = tmp_path_factory.mktemp("dropin")
    p = subprocess.run([CHECK, str(d)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    return {f[:-4]: np.load(os.path.join(d, f)) for f in os.listdir(d) if f.endswith(".npy")}


def omap(o):
    return oracle.GaussianMap(o["positions"], o["rotations"], o["colors"], o["log_scales"], o["opacity_logits"],
                              o["features"])


INTR = dict(fx=110.0, fy=110.0, cx=64.0, cy=48.0, width=128, height=96)


def oi():
    return oracle.make_intr(**INTR)


def test_render_and_backward(out):
    o = out
    q, t = o["pose"][:4], o["pose"][4:]
    ref = oracle.render(omap(o), q, t, oi(), threads=8)
    sp = ref["splats"]
    got_sp = o["splats"]
    assert np.array_equal(got_sp[:, 0], sp["source"])
    for j, f in enumerate(("x0", "x1", "y0", "y1")):
        assert np.array_equal(got_sp[:, 1 + j], sp[f]), f
    am = oracle.GaussianMap(o["positions"], o["rotations"], o["colors"], o["log_scales"], o["opacity_logits"],
                            np.abs(o["features"]))
    mag = oracle.render(am, q, t, oi(), threads=8)["query"]
    for f in ("color", "depth", "query", "alpha"):
        got = o[f].reshape(ref[f].shape)
        assert_close_floor(got, ref[f], 1e-4, f, cond=QUERY_COND * mag if f == "query" else None)
    g = oracle.render_backward(omap(o), q, t, oi(), sp, o["up_color"].reshape(96, 128, 3),
                               o["up_depth"].reshape(96, 128), o["up_query"].reshape(96, 128, -1), threads=8)
    for f in oracle.FIELDS:
        assert_close_floor(o["g_" + f].reshape(-1), getattr(g, f).reshape(-1), 1e-3, f)


def test_decoder_and_trust(out):
    o = out
    rec, att = oracle.reconstruct(o["Q"], o["atoms"], o["proj"], np.float32(2.0), want_attention=True)
    assert_close_floor(o["rec"], rec, 1e-4, "reconstruct")
    assert_close_floor(o["attention"], att, 1e-4, "attention")
    g = oracle.reconstruct_backward(o["Q"], att, o["atoms"], o["proj"], np.float32(2.0), o["dF"])
    for k, name in (("d_queries", "dg_queries"), ("d_proj", "dg_proj"), ("d_atoms", "dg_atoms")):
        assert_close_floor(o[name], g[k], 1e-3, k)
    p, tg = oracle.trust_region_penalty(o["atoms"], o["anchor"], np.float32(0.1), want_grad=True)
    assert float(o["trust"][0]) == pytest.approx(float(p), rel=1e-5)
    assert_close_floor(o["trust_grad"], tg, 1e-4, "trust grad")


def test_losses(out):
    o = out
    color = o["color"].reshape(96, 128, 3)
    depth = o["depth"].reshape(96, 128)
    alpha = o["alpha"].reshape(96, 128)
    r = oracle.rgb_loss(color, o["obs_rgb"].reshape(96, 128, 3), np.float32(0.2), np.float32(0.8))
    assert o["rgb_loss"] == pytest.approx([r["value"], r["l1"], r["ssim_loss"]], rel=2e-4)
    assert_close_floor(o["rgb_grad"].reshape(-1), r["grad"].reshape(-1), 1e-3, "rgb grad")
    d = oracle.depth_loss(depth, o["obs_depth"].reshape(96, 128), alpha)
    assert o["depth_loss"][0] == pytest.approx(float(d["value"]), rel=2e-4) and o["depth_loss"][1] == 0.0
    assert_close_floor(o["depth_grad"].reshape(-1), d["grad"].reshape(-1), 1e-5, "depth grad")
    s, sg = oracle.ssim(color, o["obs_rgb"].reshape(96, 128, 3), want_grad=True)
    assert float(o["ssim"][0]) == pytest.approx(float(s), rel=1e-5)
    assert_close_floor(o["ssim_grad"].reshape(-1), sg.reshape(-1), 1e-3, "ssim grad")
    f = oracle.feature_loss(o["rec"], o["feat_target"], o["atoms"], o["anchor"], np.float32(0.1), np.float32(0.5),
                            np.float32(0.5), np.float32(0.2))
    assert o["feature_loss"][:4] == pytest.approx([f["value"], f["cos_term"], f["l2_term"], f["trust_term"]],
                                                  rel=2e-4)
    assert_close_floor(o["feat_grad"], f["d_reconstructed"], 1e-4, "feature grad")
    assert_close_floor(o["feat_trust_grad"], f["d_atoms_trust"], 1e-4, "feature trust grad")


def test_total_objective(out):
    o = out
    frames = []
    for b in range(2):
        q, t = ((1, 0, 0, 0), (0, 0, 0)) if b == 0 else (o["pose"][:4], o["pose"][4:])
        frames.append(oracle.Frame(q, t, o["obs_rgb"].reshape(96, 128, 3), o["obs_depth"].reshape(96, 128),
                                   o[f"kf{b}_assignment"].reshape(-1), o[f"kf{b}_features"]))
    d = oracle.Dictionary(o["atoms"], o["anchor"], o["proj"], np.float32(2.0))
    oracle.set_gemm_threads(os.cpu_count() or 1)
    ref, (g, dp, da) = oracle.total_objective(omap(o), d, frames, oi(), oracle.Config(), threads=8)
    keys = ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust", "total")
    assert o["obj_loss"] == pytest.approx([ref[k] for k in keys], rel=2e-4, abs=1e-7)
    for f in oracle.FIELDS:
        assert_close_floor(o["og_" + f].reshape(-1), getattr(g, f).reshape(-1), 1e-3, f)
    assert_close_floor(o["og_proj"], dp, 1e-3, "d_proj")
    assert_close_floor(o["og_atoms"], da, 1e-3, "d_atoms")


def test_exception_contract(out):
    # render: bad intrinsics -> invalid_argument; render_backward on a moved pose -> runtime_error;
    # reconstruct: query dim -> invalid_argument; reconstruct_backward stale -> runtime_error;
    # trust / rgb / depth / feature shape mismatches -> invalid_argument; empty batch -> invalid_argument
    assert list(out["errors"]) == [1, 2, 1, 2, 1, 1, 1, 1, 1]
