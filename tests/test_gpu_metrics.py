"""Evaluation on the GPU against the oracle restatement of
proj/src/metrics.cpp and evaluate.cpp: per-row cosine terms, mIoU predictions and counts follow the
oracle's float operations exactly (counts compared ==), means over rows to double rounding."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2602_12314_b200 import _capi, api, synthetic  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return api.Context(0)


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def test_metric_cos_matches_oracle(ctx):
    g = np.random.default_rng(1)
    rec = g.standard_normal((5000, 64)).astype(np.float32)
    tgt = (rec + 0.3 * g.standard_normal(rec.shape)).astype(np.float32)
    v, fl = api.metric_cos(ctx, dev(rec), dev(tgt))
    vo, flo = oracle.metric_cos(rec, tgt)
    assert v == pytest.approx(vo, rel=1e-12) and fl == flo is False
    rec[17] = 0
    v, fl = api.metric_cos(ctx, dev(rec), dev(tgt))
    vo, flo = oracle.metric_cos(rec, tgt)
    assert v == pytest.approx(vo, rel=1e-12) and fl and flo


def test_metric_miou_counts_bit_exact(ctx):
    g = np.random.default_rng(2)
    emb = g.standard_normal((3000, 16)).astype(np.float32)
    protos = g.standard_normal((7, 16)).astype(np.float32)
    labels = g.integers(-1, 7, 3000).astype(np.int32)
    m, inter, uni = api.metric_miou(ctx, dev(emb), dev(labels), dev(protos))
    mo, io, uo = oracle.metric_miou(emb, labels, protos)
    assert np.array_equal(inter, io) and np.array_equal(uni, uo)
    assert m == pytest.approx(mo, rel=1e-14)
    with pytest.raises(_capi.InvalidArgument, match="label id out of range"):
        api.metric_miou(ctx, dev(emb), dev(np.full(3000, 7, np.int32)), dev(protos))


def test_metric_psnr_matches_oracle(ctx):
    g = np.random.default_rng(3)
    a = g.uniform(0, 1, (48, 64, 3)).astype(np.float32)
    b = (a + 0.05 * g.standard_normal(a.shape)).astype(np.float32)
    db, ex = api.metric_psnr(ctx, dev(a), dev(b))
    dbo, exo = oracle.metric_psnr(a, b)
    assert db == pytest.approx(dbo, rel=1e-12) and not ex and not exo
    assert api.metric_psnr(ctx, dev(a), dev(a)) == (100.0, True)


def test_gather_supervision_rows(ctx):
    g = np.random.default_rng(4)
    h, w, ds, df, n_set = 37, 53, 8, 24, 6
    query = g.standard_normal((h, w, ds)).astype(np.float32)
    asg = g.integers(-1, n_set, (h, w)).astype(np.int32)
    feats = g.standard_normal((n_set, df)).astype(np.float32)
    q, t, pix = api.gather_supervision(ctx, dev(query), dev(asg), dev(feats))
    sel = np.flatnonzero(asg.reshape(-1) >= 0)
    assert np.array_equal(pix.cpu().numpy(), sel)
    assert np.array_equal(q.cpu().numpy(), query.reshape(-1, ds)[sel])
    assert np.array_equal(t.cpu().numpy(), feats[asg.reshape(-1)[sel]])
    _, tn, _ = api.gather_supervision(ctx, dev(query), dev(asg), dev(feats), normalize=True)
    ref = feats[asg.reshape(-1)[sel]]
    ref = ref / np.linalg.norm(ref, axis=1, keepdims=True)
    assert np.allclose(tn.cpu().numpy(), ref, rtol=1e-6, atol=1e-7)


def test_query_map_matches_oracle(ctx):
    g = np.random.default_rng(5)
    n, ds, k, df = 2000, 8, 16, 32
    feats = g.standard_normal((n, ds)).astype(np.float32)
    atoms = g.standard_normal((k, df)).astype(np.float32)
    proj = g.standard_normal((ds, df)).astype(np.float32)
    e = g.standard_normal(df).astype(np.float32)
    s = api.query_map(ctx, dev(feats), dev(atoms), dev(proj), 2.0, dev(e)).cpu().numpy()
    so = oracle.query_scores(oracle.reconstruct(feats, atoms, proj, np.float32(2.0)), e)
    assert np.allclose(s, so, rtol=1e-4, atol=1e-5)


def test_evaluate_map_matches_oracle_pipeline(ctx):
    """evaluate_map (evaluate.cpp:10-72) on the config-0 scene: GPU render + gather + reconstruct +
    metrics against the oracle's render + reconstruct + metrics (labels = the frame's cells,
    prototypes = their embeddings)."""
    def orender(m, q, t, intr):
        om = oracle.GaussianMap(*[np.ascontiguousarray(getattr(m, f), np.float32) for f in oracle.FIELDS])
        out = oracle.render(om, q, t, oracle.make_intr(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
        return out["color"], out["depth"], out["alpha"]

    w = synthetic.make_workload(0, orender)
    fr = w.frames[0]
    gm = api.GaussianMap.from_numpy(w.map)
    intr = api.make_intrinsics(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height)
    protos = fr.features
    dframe = synthetic.Frame(fr.pose_rot, fr.pose_trans, dev(fr.rgb), dev(fr.depth), dev(fr.assignment),
                             dev(fr.features))
    dframe.labels = dev(fr.assignment)
    res = api.evaluate_map(ctx, gm, dev(w.atoms), dev(w.proj), w.temperature, [dframe], intr, prototypes=dev(protos))
    # oracle pipeline
    om = oracle.GaussianMap(*[np.ascontiguousarray(getattr(w.map, f), np.float32) for f in oracle.FIELDS])
    out = oracle.render(om, fr.pose_rot, fr.pose_trans, oracle.make_intr(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy,
                                                                        w.intr.width, w.intr.height))
    psnr = oracle.metric_psnr(out["color"], fr.rgb)[0]
    a = fr.assignment.reshape(-1)
    sel = np.flatnonzero(a >= 0)
    q = np.ascontiguousarray(out["query"].reshape(-1, out["query"].shape[-1])[sel])
    t = fr.features[a[sel]]
    t = (t / np.linalg.norm(t, axis=1, keepdims=True)).astype(np.float32)
    rec = oracle.reconstruct(q, w.atoms, w.proj, np.float32(w.temperature))
    cos = oracle.metric_cos(rec, t)[0]
    miou = oracle.metric_miou(rec, a[sel], protos)[0]
    assert res["psnr"] == pytest.approx(psnr, rel=1e-4)
    assert res["cos_loss"] == pytest.approx(cos, rel=1e-4)
    assert res["miou"] == pytest.approx(miou, abs=2e-3)
    assert res["frames"][0]["labeled_pixels"] == len(sel)
