"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the same seeded
inputs. Bars (BASELINE.json north_star / SURVEY.md §8(d)):
  - projected splats, tile lists and sort order: bit-exact;
  - rendered colour / depth / query / alpha: |a-b| <= 1e-4 * max(|b|, 1e-3 * max|b|), and
    norm-wise <= 1e-4; the query in fast mode (tensor-core sums) adds the float summation-error
    scale 2^-16 * sum_i w_i |f_i| per pixel (QUERY_COND below);
  - gradients: |a-b| <= 1e-3 * max(|b|, 1e-3 * ||b||_inf) per block (plus norm-wise);
  - decoded embeddings: per-row cosine >= 0.999.
"""
import math

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_12314_b200 import api  # noqa: E402
from paper_2602_12314_b200 import synthetic  # noqa: E402
from paper_2602_12314_b200 import _capi  # noqa: E402
from paper_2602_12314_b200._capi import StaleCache  # noqa: E402

THREADS = 8


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return api.Context(0)


def oracle_render_fn(m, q, t, intr):
    om = oracle.GaussianMap(m.positions, m.rotations, m.colors, m.log_scales, m.opacity_logits, m.features)
    oi = oracle.make_intr(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
    out = oracle.render(om, q, t, oi, threads=THREADS)
    return out["color"], out["depth"], out["alpha"]


@pytest.fixture(scope="module")
def cfg0():
    return synthetic.make_workload(0, oracle_render_fn)


def to_oracle_map(m):
    return oracle.GaussianMap(*[np.ascontiguousarray(getattr(m, f), np.float32) for f in oracle.FIELDS])


def oi(intr):
    return oracle.make_intr(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)


def gi(intr):
    return api.make_intrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)


def block_offsets(s):
    """[(begin, end)] of the 8 flat-buffer blocks (16-byte aligned; latmap_session_grad_layout)."""
    return [(o, o + n) for o, n in s.grad_blocks().values()]


def assert_close_floor(a, b, rtol, name, floor=1e-3, cond=None):
    """|a-b| <= rtol * max(|b|, floor * max|b|)  [+ cond: an extra per-element absolute allowance]."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = np.maximum(np.abs(b), floor * max(np.abs(b).max(), 1e-30))
    tol = rtol * scale if cond is None else rtol * scale + cond
    err = np.abs(a - b) / tol
    worst = err.max() if err.size else 0.0
    assert worst <= 1.0, f"{name}: max err/tol {worst:.3e} (at {np.unravel_index(err.argmax(), err.shape)})"
    if b.size:
        nrm = np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)
        assert nrm <= rtol, f"{name}: norm-wise err {nrm:.3e}"


# Fast-mode query channels are summed on the tensor cores (3xTF32: each product exact to ~2^-21,
# fp32 accumulation in a different order than the reference's sequential float loop). Where the
# features cancel, |b| is far below the summed magnitude M(p) = sum_i w_i |f_i| and BOTH float sums
# carry an absolute error of order n * 2^-24 * M(p) (n = blended splats, ~100 at config 0). The
# bound adds that error scale, QUERY_COND * M(p) with QUERY_COND = 2^-16 (n * 2^-24 for n = 256),
# to the 1e-4 relative / 1e-3 floor bar; M(p) is the oracle's render of the same map with |f|.
QUERY_COND = 2.0 ** -16


def query_magnitude(m, q, t, intr):
    am = oracle.GaussianMap(m.positions, m.rotations, m.colors, m.log_scales, m.opacity_logits,
                            np.abs(np.asarray(m.features, np.float32)))
    return oracle.render(am, q, t, oi(intr), threads=THREADS)["query"]


# ------------------------------------------------------------------------------- renderer
def test_projection_and_tiles_bit_exact(ctx, cfg0):
    w = cfg0
    om = to_oracle_map(w.map)
    ref = oracle.render(om, (1, 0, 0, 0), (0, 0, 0), oi(w.intr), threads=THREADS)
    gm = api.GaussianMap.from_numpy(w.map)
    out = api.render(ctx, gm, api.make_pose(), gi(w.intr))
    got = out.splats()
    rs = ref["splats"]
    assert len(got) == len(rs) and len(rs) > 1000
    assert np.array_equal(got["source"], rs["source"])
    for f in ("x0", "x1", "y0", "y1"):
        assert np.array_equal(got[f], rs[f]), f
    for f in ("mean", "cov_inv", "depth", "alpha"):
        assert np.array_equal(got[f].view(np.uint32), np.ascontiguousarray(rs[f]).astype(np.float32).view(np.uint32)), f
    # canonical tile lists from the reference's own splat list
    tx, ty, off, src = out.tiles()
    assert tx == math.ceil(w.intr.width / 16) and ty == math.ceil(w.intr.height / 16)
    tx0, tx1, ty0, ty1 = rs["x0"] // 16, rs["x1"] // 16, rs["y0"] // 16, rs["y1"] // 16
    order = np.lexsort((rs["source"], rs["depth"]))
    expect = [[] for _ in range(tx * ty)]
    for k in order:
        for yy in range(ty0[k], ty1[k] + 1):
            for xx in range(tx0[k], tx1[k] + 1):
                expect[yy * tx + xx].append(rs["source"][k])
    for t in range(tx * ty):
        assert np.array_equal(src[off[t]:off[t + 1]], np.asarray(expect[t], np.int32)), f"tile {t}"


@pytest.mark.parametrize("exact", [False, True])
def test_render_images_match(ctx, cfg0, exact):
    w = cfg0
    ref = oracle.render(to_oracle_map(w.map), (1, 0, 0, 0), (0, 0, 0), oi(w.intr), threads=THREADS)
    ctx.set_exact_blend(exact)
    try:
        out = api.render(ctx, api.GaussianMap.from_numpy(w.map), api.make_pose(), gi(w.intr))
    finally:
        ctx.set_exact_blend(False)
    mag = query_magnitude(to_oracle_map(w.map), (1, 0, 0, 0), (0, 0, 0), w.intr)
    for f in ("color", "depth", "query", "alpha"):
        g = getattr(out, f).cpu().numpy()
        # exact mode: the tight bar alone; fast mode's query: plus the summation-error scale
        cond = QUERY_COND * mag if (f == "query" and not exact) else None
        assert_close_floor(g, ref[f], 1e-4, f, floor=1e-3, cond=cond)
        if f == "query":
            e = np.abs(g.astype(np.float64) - ref[f]) / np.maximum(mag, 1e-30)
            print(f"query (exact={exact}): max |a-b| / M(p) = {e.max():.3e} (bound {QUERY_COND:.3e})")
        same = np.mean(g.view(np.uint32) == ref[f].astype(np.float32).view(np.uint32))
        if exact:  # exact mode: libm expf and the reference's op order -> the reference's bits
            assert same > 0.999, f"{f}: only {same:.5f} of values bit-identical"
        elif f == "alpha":  # fast mode: exp on the SFU (ex2.approx): alpha within ~1e-6 relative
            np.testing.assert_allclose(g, ref[f], rtol=1e-5, atol=1e-6)


def test_render_posed_camera(ctx):
    rng = np.random.default_rng(5)
    m = synthetic.random_map(rng, 5000, (-2, -1.5, 1), (2, 1.5, 6), 8)
    intr = synthetic.Intr(200.0, 200.0, 96.0, 64.0, 192, 128)
    q = synthetic.yaw_quat(0.07)
    t = (0.05, -0.02, 0.1)
    ref = oracle.render(to_oracle_map(m), q, t, oi(intr), threads=THREADS)
    out = api.render(ctx, api.GaussianMap.from_numpy(m), api.make_pose(q, t), gi(intr))
    assert np.array_equal(out.splats()["source"], ref["splats"]["source"])
    mag = query_magnitude(to_oracle_map(m), q, t, intr)
    for f in ("color", "depth", "query", "alpha"):
        assert_close_floor(getattr(out, f).cpu().numpy(), ref[f], 1e-4, f, floor=1e-3,
                           cond=QUERY_COND * mag if f == "query" else None)


def test_render_edge_cases(ctx):
    intr = synthetic.Intr(100.0, 100.0, 32.0, 24.0, 64, 48)
    # empty map -> zero images (test_render.cpp:112-118)
    empty = synthetic.HostMap(*[np.zeros(s, np.float32) for s in ((0, 3), (0, 4), (0, 3), (0, 3), (0,), (0, 3))])
    out = api.render(ctx, api.GaussianMap.from_numpy(empty), api.make_pose(), gi(intr))
    assert float(out.alpha.abs().max()) == 0.0 and float(out.color.abs().max()) == 0.0
    # single opaque Gaussian (test_render.cpp:70-89) in float
    one = synthetic.HostMap(np.array([[0, 0, 1.0]], np.float32), np.array([[1.0, 0, 0, 0]], np.float32),
                            np.array([[0.2, 0.6, 0.9]], np.float32), np.full((1, 3), math.log(0.2), np.float32),
                            np.array([40.0], np.float32), np.array([[1.0, 2, 3, 4]], np.float32))
    out = api.render(ctx, api.GaussianMap.from_numpy(one), api.make_pose(), gi(intr))
    assert out.alpha[24, 32].item() == pytest.approx(0.999, rel=1e-6)
    assert out.query[24, 32, 3].item() == pytest.approx(4 * 0.999, rel=1e-6)
    # invalid intrinsics -> std::invalid_argument
    with pytest.raises(ValueError):
        api.render(ctx, api.GaussianMap.from_numpy(one), api.make_pose(), api.make_intrinsics(0, 0, 0, 0, 4, 4))
    # project_gaussian KATs (test_render.cpp:38-68)
    r = api.project_gaussian(ctx, (0, 0, 1), (1, 0, 0, 0), [math.log(0.05)] * 3, 0.0, api.make_pose(), gi(intr))
    assert r[0][0] == pytest.approx(32.0) and r[0][1] == pytest.approx(24.0) and r[2] == pytest.approx(1.0)
    r = api.project_gaussian(ctx, (0, 0, 2.0), (1, 0, 0, 0), [math.log(0.08)] * 3, 0.0, api.make_pose(), gi(intr))
    assert r[1][0, 0] == pytest.approx((100 * 0.08 / 2) ** 2 + 0.3, rel=1e-5)
    assert api.project_gaussian(ctx, (0, 0, -0.5), (1, 0, 0, 0), [math.log(0.05)] * 3, 0, api.make_pose(),
                                gi(intr)) is None


def test_render_backward_matches(ctx):
    rng = np.random.default_rng(7)
    m = synthetic.random_map(rng, 3000, (-2, -1.5, 1), (2, 1.5, 6), 16)
    m.log_scales = (m.log_scales + 1.0).astype(np.float32)  # larger footprints: more overlap
    intr = synthetic.Intr(160.0, 160.0, 64.0, 48.0, 128, 96)
    q, t = synthetic.yaw_quat(0.03), (0.02, 0.0, -0.05)
    h, w_ = intr.height, intr.width
    uc = rng.uniform(-1, 1, (h, w_, 3)).astype(np.float32)
    ud = rng.uniform(-1, 1, (h, w_)).astype(np.float32)
    uq = rng.uniform(-1, 1, (h, w_, 16)).astype(np.float32)
    om = to_oracle_map(m)
    ref = oracle.render(om, q, t, oi(intr), threads=THREADS)
    rg = oracle.render_backward(om, q, t, oi(intr), ref["splats"], uc, ud, uq, threads=THREADS)
    gm = api.GaussianMap.from_numpy(m)
    pose = api.make_pose(q, t)
    out = api.render(ctx, gm, pose, gi(intr))
    dev = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    g = api.render_backward(ctx, gm, pose, gi(intr), out, dev(uc), dev(ud), dev(uq))
    for f in oracle.FIELDS:
        assert_close_floor(getattr(g, f).cpu().numpy(), getattr(rg, f), 1e-3, f)
    # stale cache (test_render.cpp:212-221)
    gm2 = api.GaussianMap.from_numpy(synthetic.random_map(rng, 3001, (-2, -1.5, 1), (2, 1.5, 6), 16))
    with pytest.raises(StaleCache):
        api.render_backward(ctx, gm2, pose, gi(intr), out, dev(uc), dev(ud), dev(uq))


# ------------------------------------------------------------------------------- decoder / losses
def test_reconstruct_and_backward(ctx):
    rng = np.random.default_rng(11)
    n, ds, k, df = 3000, 16, 64, 96
    q = rng.standard_normal((n, ds)).astype(np.float32)
    atoms = rng.standard_normal((k, df)).astype(np.float32)
    proj = (rng.standard_normal((ds, df)) * 0.2).astype(np.float32)
    tau = 4.0
    f_ref, att_ref = oracle.reconstruct(q, atoms, proj, tau, want_attention=True)
    dev = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    f, att = api.reconstruct(ctx, dev(q), dev(atoms), dev(proj), tau, want_attention=True)
    f = f.cpu().numpy()
    cos = (f * f_ref).sum(1) / (np.linalg.norm(f, axis=1) * np.linalg.norm(f_ref, axis=1))
    assert cos.min() >= 0.999999
    assert_close_floor(f, f_ref, 1e-3, "reconstruct")  # spec: cosine >= 0.999 (checked above)
    up = rng.standard_normal((n, df)).astype(np.float32)
    gr = oracle.reconstruct_backward(q, att_ref, atoms, proj, tau, up)
    gg = api.reconstruct_backward(ctx, dev(q), att, dev(atoms), dev(proj), tau, dev(up))
    for key in ("d_queries", "d_proj", "d_atoms"):
        assert_close_floor(gg[key].cpu().numpy(), gr[key], 1e-3, key)
    with pytest.raises(ValueError):
        api.reconstruct(ctx, dev(q[:, :7].copy()), dev(atoms), dev(proj), tau)


def test_trust_region_and_ssim(ctx):
    rng = np.random.default_rng(12)
    anchor = rng.standard_normal((64, 128)).astype(np.float32)
    atoms = (anchor + rng.standard_normal((64, 128)) * 0.02).astype(np.float32)
    dev = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    p, g = api.trust_region_penalty(ctx, dev(atoms), dev(anchor), 0.2, want_grad=True)
    pr, grf = oracle.trust_region_penalty(atoms, anchor, np.float32(0.2), want_grad=True)
    assert p == pytest.approx(pr, rel=1e-5, abs=1e-6)
    assert_close_floor(g.cpu().numpy(), grf, 1e-4, "trust grad")
    a = rng.random((48, 64, 3)).astype(np.float32)
    b = rng.random((48, 64, 3)).astype(np.float32)
    v, da = api.ssim(ctx, dev(a), dev(b), want_grad=True)
    vr, dar = oracle.ssim(a, b, want_grad=True)
    assert v == pytest.approx(vr, rel=1e-5, abs=1e-6)
    assert_close_floor(da.cpu().numpy(), dar, 1e-3, "ssim grad")
    s = rng.random((6, 7, 2)).astype(np.float32)  # whole-image fallback
    assert api.ssim(ctx, dev(s), dev(s)) == pytest.approx(1.0, abs=1e-5)


def test_adam_bit_exact(ctx):
    rng = np.random.default_rng(13)
    p = rng.standard_normal(10000).astype(np.float32)
    st_ref = oracle.AdamState(np.zeros_like(p), np.zeros_like(p))
    pr = p.copy()
    dev = lambda a: torch.as_tensor(a, device="cuda")  # noqa: E731
    pg = dev(p)
    st = api.AdamState(torch.zeros_like(pg), torch.zeros_like(pg))
    for it in range(5):
        g = rng.standard_normal(10000).astype(np.float32)
        oracle.adam_step(pr, g, st_ref, np.float32(0.01))
        api.adam_step(ctx, pg, dev(g), st, 0.01)
    assert np.array_equal(pg.cpu().numpy().view(np.uint32), pr.view(np.uint32))
    assert st.step == st_ref.step == 5
    g = np.ones_like(p)
    g[3] = np.nan
    assert not api.adam_step(ctx, pg, dev(g), st, 0.01)
    assert st.skipped == 1


# ------------------------------------------------------------------------------- full step
def make_session(ctx, w, **over):
    cfg = api.default_config(**{**w.lambdas, **over})
    s = api.Session(ctx, cfg, w.map.n, w.map.features.shape[1], w.atoms.shape[0], w.atoms.shape[1], gi(w.intr))
    s.set_map(w.map)
    s.set_dictionary(w.atoms, w.anchor, w.proj)
    s.set_frames(w.frames)
    s.set_batch(len(w.frames))
    return s


def oracle_cfg(w):
    c = oracle.Config(lambda_l2=w.lambdas["lambda_l2"], lambda_i2=w.lambdas["lambda_i2"],
                      lambda_trust=w.lambdas["lambda_trust"])
    return c


def oracle_frames(w):
    return [oracle.Frame(f.pose_rot, f.pose_trans, f.rgb, f.depth, f.assignment.reshape(-1), f.features)
            for f in w.frames]


def dict_grads_f64(w, query_f32, lam):
    """Ground truth for d_proj / d_atoms: the reference decoder algebra in double on the (bit-exact
    float) rendered queries, scaled as total_objective does (objective.cpp:130-135,176-185)."""
    f64 = np.float64
    q = query_f32.reshape(-1, query_f32.shape[-1]).astype(f64)
    fr = w.frames[0]
    a = fr.assignment.reshape(-1)
    sup = a >= 0
    q = np.ascontiguousarray(q[sup])
    tgt = np.ascontiguousarray(fr.features.astype(f64)[a[sup]])
    atoms, anchor, proj = (x.astype(f64) for x in (w.atoms, w.anchor, w.proj))
    tau = f64(np.float32(w.temperature))
    rec, att = oracle.reconstruct(q, atoms, proj, tau, want_attention=True)
    fl = oracle.feature_loss(rec, tgt, atoms, anchor, f64(np.float32(0.1)), f64(np.float32(0.5)),
                             f64(np.float32(lam["lambda_l2"])), f64(np.float32(lam["lambda_trust"])), True)
    g = oracle.reconstruct_backward(q, att, atoms, proj, tau, fl["d_reconstructed"])
    lf = f64(np.float32(5.0))
    _, tg = oracle.trust_region_penalty(atoms, anchor, f64(np.float32(0.1)), want_grad=True)
    return lf * g["d_proj"], lf * g["d_atoms"] + lf * f64(np.float32(lam["lambda_trust"])) * tg


def test_session_objective_config0(ctx, cfg0):
    w = cfg0
    s = make_session(ctx, w)
    loss = s.objective(want_grad=True)
    d = oracle.Dictionary(w.atoms.copy(), w.anchor.copy(), w.proj.copy(), np.float32(w.temperature))
    ref, (g, dp, da) = oracle.total_objective(to_oracle_map(w.map), d, oracle_frames(w), oi(w.intr), oracle_cfg(w),
                                              threads=THREADS)
    for key in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust", "total"):
        assert loss[key] == pytest.approx(ref[key], rel=2e-4, abs=1e-6), key
    assert loss["supervised_rows"] == ref["supervised_rows"]
    gb = s.grad_buffer().cpu().numpy()
    n, ds = w.map.n, w.map.features.shape[1]
    offs = block_offsets(s)
    # map gradients: against the fp32 reference path (identical render decisions)
    blocks = [g.positions, g.rotations, g.colors, g.log_scales, g.opacity_logits, g.features]
    for i, (name, ref_b) in enumerate(zip(oracle.FIELDS, blocks)):
        assert_close_floor(gb[offs[i][0]:offs[i][1]], ref_b.reshape(-1), 1e-3, name)
    # dictionary gradients: sums over 76.8k rows; judged against the double-precision truth on the
    # same rendered queries (the fp32 reference itself sits ~1e-3 away from it on small entries)
    _, _, q_img, _ = s.frame_images(0)
    tp, ta = dict_grads_f64(w, q_img.cpu().numpy(), w.lambdas)
    assert_close_floor(gb[offs[6][0]:offs[6][1]], tp.reshape(-1), 1e-3, "d_proj")
    assert_close_floor(gb[offs[7][0]:offs[7][1]], ta.reshape(-1), 1e-3, "d_atoms")
    # and the fp32 reference agrees with the GPU norm-wise
    for name, got, r in (("d_proj", gb[offs[6][0]:offs[6][1]], dp), ("d_atoms", gb[offs[7][0]:offs[7][1]], da)):
        nrm = np.linalg.norm(got - r.reshape(-1)) / np.linalg.norm(r)
        assert nrm < 1e-3, (name, nrm)


def test_session_step_config0_adam(ctx, cfg0):
    w = cfg0
    s = make_session(ctx, w)
    s.step(read=True)
    got = s.get_map()
    atoms, proj = s.get_dictionary()
    om = to_oracle_map(w.map)
    d = oracle.Dictionary(w.atoms.copy(), w.anchor.copy(), w.proj.copy(), np.float32(w.temperature))
    cfg = oracle_cfg(w)
    _, (g, dp, da) = oracle.total_objective(om, d, oracle_frames(w), oi(w.intr), cfg, threads=THREADS)
    opt = oracle.MapOptimizer()
    opt.step_map(om, g, cfg)
    opt.step_dict(d, dp, da, cfg)
    # first Adam step moves each coordinate by ~lr * sign(g): compare within a 1e-5 relative band
    # except where the reference gradient is ~0 (sign not determined at fp32).
    for name, a, b, gref, lr in [("positions", got["positions"], om.positions, g.positions, 1e-4),
                                 ("colors", got["colors"], om.colors, g.colors, 2.5e-3),
                                 ("features", got["features"], om.features, g.features, 2.5e-3),
                                 ("atoms", atoms, d.atoms, da, 1e-2), ("proj", proj, d.proj, dp, 1e-2)]:
        diff = np.abs(a - b)
        tiny = np.abs(gref) <= 1e-3 * np.abs(gref).max()
        bad = (diff > 1e-5 * np.maximum(np.abs(b), 1.0)) & ~tiny
        assert bad.mean() < 1e-3, f"{name}: {bad.mean():.2e} of coordinates moved differently"
        assert diff.max() <= 2.0 * lr + 1e-6, name
    nq = np.linalg.norm(got["rotations"], axis=1)
    assert np.abs(nq - 1).max() < 1e-6


# ------------------------------------------------------------------------------- Stage II / row sets
def _moved_like(name, a, b, gref, lr, steps, frac=1e-2):
    """Adam moves each coordinate by at most ~lr per step; coordinates whose reference gradient is
    not ~0 must agree within a 1e-5 relative band."""
    diff = np.abs(a - b)
    tiny = np.abs(gref) <= 1e-3 * np.abs(gref).max()
    bad = (diff > 1e-5 * np.maximum(np.abs(b), 1.0)) & ~tiny
    assert bad.mean() < frac, f"{name}: {bad.mean():.2e} of coordinates moved differently"
    assert diff.max() <= 2.0 * lr * steps + 1e-6, name


def test_stage2_render_cache_bit_identical(ctx, cfg0):
    """ObjectiveOptions::cached_renders (objective.cpp:88-96): with the map unchanged, the cached
    objective equals a freshly rendered one bit for bit, and step_dict leaves the map untouched."""
    w = cfg0
    s = make_session(ctx, w)
    s.step(read=False)
    fresh = s.objective_ex(want_grad=False, map_grads=False, use_cached_renders=False)
    cached = s.objective_ex(want_grad=False, map_grads=False, use_cached_renders=True)
    for k in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust", "total"):
        assert cached[k] == fresh[k], k
    before = s.get_map()
    s.step_dict(read=False)
    s.step_dict(read=True)
    after = s.get_map()
    for f in oracle.FIELDS:
        assert np.array_equal(before[f], after[f]), f


def test_stage2_step_dict_matches_oracle(ctx, cfg0):
    """Stage I then two Stage II iterations (pipeline.cpp:236-259) against the oracle pipeline."""
    w = cfg0
    s = make_session(ctx, w)
    s.step(read=False)
    l2 = [s.step_dict(read=True) for _ in range(2)]
    atoms, proj = s.get_dictionary()
    om = to_oracle_map(w.map)
    d = oracle.Dictionary(w.atoms.copy(), w.anchor.copy(), w.proj.copy(), np.float32(w.temperature))
    cfg = oracle_cfg(w)
    opt = oracle.MapOptimizer()
    _, (g, dp, da) = oracle.total_objective(om, d, oracle_frames(w), oi(w.intr), cfg, threads=THREADS)
    opt.step_map(om, g, cfg)
    opt.step_dict(d, dp, da, cfg)
    for _ in range(2):
        ref, (_, dp, da) = oracle.total_objective(om, d, oracle_frames(w), oi(w.intr), cfg, threads=THREADS,
                                                  map_grads=False)
        opt.step_dict(d, dp, da, cfg)
    assert opt.states["proj"].step == 3 and opt.states["positions"].step == 1
    got = s.get_map()
    _moved_like("positions", got["positions"], om.positions, g.positions, 1e-4, 1)
    _moved_like("atoms", atoms, d.atoms, da, 1e-2, 3)
    _moved_like("proj", proj, d.proj, dp, 1e-2, 3)
    # the loss reported by the last Stage II call is that of the dictionary before its update
    assert l2[-1]["total"] == pytest.approx(ref["total"], rel=1e-3)


def test_export_import_rows_keep_and_append(ctx, cfg0):
    """Active-set row changes: keep_map_rows compaction of the Adam moments plus zero-moment
    newborns (pipeline.cpp:97-104, adam.hpp:18-29), checked through the next Adam step."""
    w = cfg0
    s = make_session(ctx, w)
    s.step(read=False)
    rows = s.export_rows()
    m0 = s.get_map()
    flat = np.concatenate([m0["positions"], m0["rotations"], m0["colors"], m0["log_scales"],
                           m0["opacity_logits"][:, None], m0["features"]], axis=1)
    assert np.array_equal(rows.cpu().numpy(), flat)
    rng = np.random.default_rng(7)
    kept = rng.random(w.map.n) < 0.8
    extra = synthetic.random_map(rng, 1000, (-2, -1.5, 1), (2, 1.5, 6), w.map.features.shape[1])
    extra_rows = np.concatenate([extra.positions, extra.rotations, extra.colors, extra.log_scales,
                                 extra.opacity_logits[:, None], extra.features], axis=1).astype(np.float32)
    new_rows = np.concatenate([flat[kept], extra_rows], axis=0)
    s.import_rows(torch.from_numpy(new_rows).cuda(), kept=kept)
    assert s.n == new_rows.shape[0]
    got = s.get_map()
    assert np.array_equal(got["positions"], new_rows[:, :3]) and np.array_equal(got["features"], new_rows[:, 14:])
    s.step(read=False)
    after = s.get_map()
    # oracle: same Stage-I step, moments compacted (kept rows) and zero for the appended rows
    om = to_oracle_map(w.map)
    d = oracle.Dictionary(w.atoms.copy(), w.anchor.copy(), w.proj.copy(), np.float32(w.temperature))
    cfg = oracle_cfg(w)
    opt = oracle.MapOptimizer()
    _, (g, dp, da) = oracle.total_objective(om, d, oracle_frames(w), oi(w.intr), cfg, threads=THREADS)
    opt.step_map(om, g, cfg)
    opt.step_dict(d, dp, da, cfg)
    nm = oracle.GaussianMap(*[np.ascontiguousarray(x, np.float32) for x in (
        new_rows[:, :3], new_rows[:, 3:7], new_rows[:, 7:10], new_rows[:, 10:13], new_rows[:, 13], new_rows[:, 14:])])
    for name in oracle.FIELDS:
        st = opt.states[name]
        pad = [(0, 1000)] + [(0, 0)] * (st.m.ndim - 1)
        st.m = np.ascontiguousarray(np.pad(st.m[kept], pad))
        st.v = np.ascontiguousarray(np.pad(st.v[kept], pad))
    _, (g2, dp2, da2) = oracle.total_objective(nm, d, oracle_frames(w), oi(w.intr), cfg, threads=THREADS)
    opt.step_map(nm, g2, cfg)
    _moved_like("positions", after["positions"], nm.positions, g2.positions, 1e-4, 2)
    _moved_like("features", after["features"], nm.features, g2.features, 2.5e-3, 2)
    _moved_like("colors", after["colors"], nm.colors, g2.colors, 2.5e-3, 2)


@pytest.mark.parametrize("det", [False, True])
def test_session_segment_supervision_config0(ctx, cfg0, det):
    """feature_supervision = "segment" (objective.cpp:37-64, 147-157): queries pooled per present
    assignment row, the row gradient shared equally by the segment's pixels (also in the
    deterministic mode, whose pooling sums each segment in raster order)."""
    w = cfg0
    s = make_session(ctx, w, segment_mode=1, decoder_precision=0)
    ctx.set_deterministic(det)
    try:
        loss = s.objective(want_grad=True)
    finally:
        ctx.set_deterministic(False)
    d = oracle.Dictionary(w.atoms.copy(), w.anchor.copy(), w.proj.copy(), np.float32(w.temperature))
    cfg = oracle_cfg(w)
    cfg.segment_mode = True
    ref, (g, dp, da) = oracle.total_objective(to_oracle_map(w.map), d, oracle_frames(w), oi(w.intr), cfg,
                                              threads=THREADS)
    assert loss["supervised_rows"] == ref["supervised_rows"] == len(np.unique(w.frames[0].assignment[
        w.frames[0].assignment >= 0]))
    for key in ("l_rgb", "l_depth", "l_cos", "l_l2", "l_trust", "total"):
        assert loss[key] == pytest.approx(ref[key], rel=2e-4, abs=1e-6), key
    gb = s.grad_buffer().cpu().numpy()
    n, ds = w.map.n, w.map.features.shape[1]
    offs = block_offsets(s)
    blocks = [g.positions, g.rotations, g.colors, g.log_scales, g.opacity_logits, g.features]
    for i, (name, ref_b) in enumerate(zip(oracle.FIELDS, blocks)):
        assert_close_floor(gb[offs[i][0]:offs[i][1]], ref_b.reshape(-1), 1e-3, name)
    for name, got, r in (("d_proj", gb[offs[6][0]:offs[6][1]], dp), ("d_atoms", gb[offs[7][0]:offs[7][1]], da)):
        assert_close_floor(got, r.reshape(-1), 1e-3, name)


def test_graph_replay_matches_direct_steps(ctx, cfg0):
    """Steps replayed from the captured CUDA graph equal directly launched steps (up to the
    run-to-run rounding of the atomic gradient sums), and a pose change re-captures."""
    w = cfg0
    a = make_session(ctx, w)
    b = make_session(ctx, w)
    b.set_graphs(False)
    for _ in range(3):
        la = a.step(read=True)
        lb = b.step(read=True)
    assert la["total"] == pytest.approx(lb["total"], rel=1e-5)
    ma, mb = a.get_map(), b.get_map()
    # Adam normalises each update by sqrt(v): a parameter whose gradient is ~0 moves by about
    # lr * sign(g) per step, so atomic-order noise can flip a handful of such updates. Everything
    # else must agree to float rounding.
    lr_max = 3 * 2 * max(w_lr for w_lr in (a.cfg.lr_position, a.cfg.lr_rotation, a.cfg.lr_color, a.cfg.lr_log_scale,
                                           a.cfg.lr_opacity, a.cfg.lr_feature))
    for f in oracle.FIELDS:
        bad = ~np.isclose(ma[f], mb[f], rtol=1e-5, atol=1e-6)
        assert bad.mean() < 1e-3, (f, int(bad.sum()))
        assert np.abs(ma[f] - mb[f]).max() <= lr_max * max(1.0, a.cfg.scene_extent), f
    # move the camera: the graph must not replay the old pose
    fr = w.frames[0]
    moved = synthetic.Frame(synthetic.yaw_quat(0.05), (0.02, 0.0, 0.0), fr.rgb, fr.depth, fr.assignment, fr.features)
    a.set_frames([moved])
    b.set_frames([moved])
    la, lb = a.step(read=True), b.step(read=True)
    assert la["total"] == pytest.approx(lb["total"], rel=1e-5)


def test_seed_gaussians_candidates_and_append(ctx, cfg0):
    """seed_gaussians (pipeline.cpp:39-73): stride-2 pixels with observed depth whose render leaves
    them uncovered (alpha < 0.5) or misplaced (|depth error| > 0.1), in raster order, restated in
    numpy float32 with the reference's op order; then append_newborns with zero moments."""
    w = cfg0
    s = make_session(ctx, w)
    s.step(read=False)  # the map moved: seeding renders it again
    rows = s.seed_candidates(0).cpu().numpy()
    color, depth, _, alpha = [x.cpu().numpy() for x in s.frame_images(0)]
    fr = w.frames[0]
    f32 = np.float32
    intr = w.intr
    R = oracle.quat_to_rot(fr.pose_rot, np.float32)
    t = np.asarray(fr.pose_trans, f32)
    exp = []
    for y in range(0, intr.height, 2):
        for x in range(0, intr.width, 2):
            z = fr.depth[y, x]
            if not z > 0:
                continue
            if not (alpha[y, x] < f32(0.5) or abs(f32(depth[y, x] - z)) > f32(0.1)):
                continue
            pc = [f32(f32(f32(f32(x) - f32(intr.cx)) / f32(intr.fx)) * z),
                  f32(f32(f32(f32(y) - f32(intr.cy)) / f32(intr.fy)) * z), z]
            pos = [f32(f32(f32(R[k, 0] * pc[0]) + f32(R[k, 1] * pc[1])) + f32(R[k, 2] * pc[2])) + t[k]
                   for k in range(3)]
            ls = f32(np.log(np.float64(f32(f32(z / f32(intr.fx)) * f32(2.0)))))
            exp.append(pos + [1, 0, 0, 0] + list(fr.rgb[y, x]) + [ls, ls, ls, 0] + [0] * w.map.features.shape[1])
    exp = np.asarray(exp, f32)
    assert rows.shape == exp.shape and rows.shape[0] > 0
    assert np.array_equal(rows, exp)
    n0 = s.n
    feats = np.random.default_rng(3).normal(0, 0.01, (rows.shape[0], w.map.features.shape[1])).astype(f32)
    s.append_rows(torch.from_numpy(rows).cuda(), feats)
    assert s.n == n0 + rows.shape[0]
    m = s.get_map()
    assert np.array_equal(m["positions"][n0:], rows[:, :3]) and np.array_equal(m["features"][n0:], feats)
    assert np.isfinite(s.step(read=True)["total"])


def test_assignment_out_of_range_is_reported(ctx, cfg0):
    """gather_supervision (objective.cpp:16-35) rejects an assignment >= n_set. The pixel-mode scan
    runs on the device behind the keyframe upload, so the objective call that reads the loss
    raises (the reference throws from inside total_objective); a valid batch afterwards works."""
    import copy
    w = cfg0
    bad = copy.deepcopy(w.frames[0])
    bad.assignment = bad.assignment.copy()
    bad.assignment.reshape(-1)[17] = bad.features.shape[0]  # == n_set: out of range
    s = make_session(ctx, w)
    s.set_frames([bad])
    with pytest.raises(_capi.InvalidArgument, match="assignment out of range"):
        s.objective(want_grad=True)
    s.set_frames(w.frames)
    loss = s.objective(want_grad=True)
    assert np.isfinite(loss["total"]) and loss["supervised_rows"] == int((w.frames[0].assignment >= 0).sum())


def test_tile_list_overflow_is_recovered(ctx, cfg0):
    """Tile-pair buffers are sized by the first step; a map whose splats grow far larger overflows
    them inside the captured (multi-stream) step. The step must detect it, discard the partial
    step (Adam skipped), grow the lists and re-run: same loss and map as a fresh session."""
    import copy
    w = cfg0
    big = copy.deepcopy(w.map)
    big.log_scales = (big.log_scales + 1.5).astype(np.float32)  # ~4.5x larger footprints
    a = make_session(ctx, w)
    a.step(read=True)  # sizes the buffers for the small splats
    a.set_map(big)
    a.set_dictionary(w.atoms, w.anchor, w.proj)  # undo the first step's dictionary update
    la = a.objective(want_grad=True)
    b = make_session(ctx, w)
    b.set_map(big)
    lb = b.objective(want_grad=True)
    for k in ("l_rgb", "l_depth", "l_cos", "total"):
        assert la[k] == pytest.approx(lb[k], rel=1e-5), (k, la[k], lb[k])
    ga, gb = a.grad_buffer().cpu().numpy(), b.grad_buffer().cpu().numpy()
    assert np.linalg.norm(ga - gb) <= 1e-4 * np.linalg.norm(gb)
    la2 = a.step(read=True)  # and through the captured step
    lb2 = b.step(read=True)
    assert la2["total"] == pytest.approx(lb2["total"], rel=1e-5)


def test_objective_graph_matches_direct(ctx, cfg0):
    """latmap_session_objective replays a captured objective-only graph once the tile lists are
    sized (the multi-GPU step: objective -> all-reduce -> apply); it equals the direct launches."""
    w = cfg0
    a = make_session(ctx, w)
    b = make_session(ctx, w)
    b.set_graphs(False)
    for _ in range(3):  # first call sizes (direct), then capture, then replay
        la = a.objective(want_grad=True)
        lb = b.objective(want_grad=True)
        assert la["total"] == pytest.approx(lb["total"], rel=1e-6)
        ga, gb = a.grad_buffer().cpu().numpy(), b.grad_buffer().cpu().numpy()
        assert np.linalg.norm(ga - gb) <= 1e-5 * np.linalg.norm(gb)
    a.apply()
    b.apply()
    la, lb = a.objective(want_grad=True), b.objective(want_grad=True)
    assert la["total"] == pytest.approx(lb["total"], rel=1e-4)


def test_objective_ragged_multiframe_unsupervised(ctx):
    """Ragged image (70 x 52: partial tiles on both edges), two keyframes through the multi-stream
    pipeline, the second with no supervised pixel (decoder rows all masked, n_sup = 0): objective
    and gradients against the oracle's total_objective."""
    def orender(m, q, t, intr):
        om = oracle.GaussianMap(*[np.ascontiguousarray(getattr(m, f), np.float32) for f in oracle.FIELDS])
        out = oracle.render(om, q, t, oracle.make_intr(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
        return out["color"], out["depth"], out["alpha"]

    w = synthetic.make_workload(0, orender, scale=0.22)
    assert w.intr.width % 16 and w.intr.height % 16
    f0 = w.frames[0]
    f1 = synthetic.Frame(synthetic.yaw_quat(0.03), (0.01, 0.0, 0.0), f0.rgb, f0.depth,
                         np.full_like(f0.assignment, -1), f0.features)
    w.frames = [f0, f1]
    s = make_session(ctx, w)
    loss = s.objective(want_grad=True)
    loss = s.objective(want_grad=True)  # second call: the captured objective graph
    d = oracle.Dictionary(w.atoms.copy(), w.anchor.copy(), w.proj.copy(), np.float32(w.temperature))
    ref, (g, dp, da) = oracle.total_objective(to_oracle_map(w.map), d, oracle_frames(w), oi(w.intr), oracle_cfg(w),
                                              threads=THREADS)
    for key in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust", "total"):
        assert loss[key] == pytest.approx(ref[key], rel=2e-4, abs=1e-6), key
    assert loss["supervised_rows"] == ref["supervised_rows"]
    gb = s.grad_buffer().cpu().numpy()
    n, ds = w.map.n, w.map.features.shape[1]
    offs = block_offsets(s)
    blocks = [g.positions, g.rotations, g.colors, g.log_scales, g.opacity_logits, g.features]
    for i, (name, ref_b) in enumerate(zip(oracle.FIELDS, blocks)):
        assert_close_floor(gb[offs[i][0]:offs[i][1]], ref_b.reshape(-1), 1e-3, name)
