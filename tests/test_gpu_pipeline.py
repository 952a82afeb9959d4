"""The pipeline around the step (proj/src/pipeline.cpp:106-330) on the
GPU: ``api.Pipeline`` (csrc/pipeline.cu) against a test-side composition of the same keyframe
loop written from pipeline.cpp over the already oracle-pinned primitives (Session, Store,
stream k-means, seeding, sync). Both consume a std::mt19937_64 of the same seed in the
reference's order. The test side uses tests/native/stdrng.cpp, libstdc++'s own distributions.

Counts must agree exactly: seeded rows, active and global sizes, sync statistics and ActiveSet
origins. Losses and the final map, dictionary and store agree to float noise. The step's
gradient reductions use float atomics, so two runs are not bitwise identical; small learning
rates keep that noise away from the seeding thresholds."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_12314_b200 import api, lamt, pipeline as pl  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return api.Context(0)


@pytest.fixture(scope="module")
def stdrng(tmp_path_factory):
    so = tmp_path_factory.mktemp("rng") / "libstdrng.so"
    subprocess.run(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", os.path.join(HERE, "native", "stdrng.cpp"), "-o",
                    str(so)], check=True)
    L = C.CDLL(str(so))
    L.rng_new.restype = C.c_void_p
    L.rng_new.argtypes = [C.c_uint64]
    L.rng_uniform01.restype = C.c_double
    L.rng_uniform01.argtypes = [C.c_void_p]
    L.rng_normal.argtypes = [C.c_void_p, C.c_float, C.c_int64, C.c_void_p]
    L.rng_sample_history.restype = C.c_int64
    L.rng_sample_history.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p]
    return L


W, H = 64, 48


def make_scene(ctx, nframes=7, seed=0, ed=32, n_set=6):
    """Frames rendered from a random ground-truth map along a 0.3 m/frame walk."""
    g = np.random.default_rng(seed)
    n = 3000
    pos = np.stack([g.uniform(-2, 2, n), g.uniform(-1.5, 1.5, n), g.uniform(2, 5, n)], 1)
    q = g.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    truth = api.GaussianMap(*[torch.as_tensor(np.ascontiguousarray(a, np.float32), device="cuda") for a in (
        pos, q, g.uniform(0, 1, (n, 3)), g.normal(-2.5, 0.3, (n, 3)), g.normal(1.0, 0.5, n), g.standard_normal((n, 4)))])
    intr = api.make_intrinsics(60.0, 60.0, 32.0, 24.0, W, H)
    frames = []
    for f in range(nframes):
        rot, trans = (1.0, 0.0, 0.0, 0.0), (0.3 * f, 0.05 * f, 0.0)
        out = api.render(ctx, truth, api.make_pose(rot, trans), intr)
        dep = out.depth.cpu().numpy()
        dep[out.alpha.cpu().numpy() < 0.3] = 0  # holes: no observed depth
        seeds = g.random((n_set, 2)) * np.array([W, H])
        ys, xs = np.mgrid[0:H, 0:W]
        d = (xs[..., None] - seeds[:, 0]) ** 2 + (ys[..., None] - seeds[:, 1]) ** 2
        asg = np.argmin(d, axis=2).astype(np.int32)
        asg[::7, ::5] = -1
        feats = g.standard_normal((n_set, ed)).astype(np.float32) * 2.0
        frames.append(lamt.Keyframe(rot, trans, out.color.cpu().numpy(), dep, asg, feats, frame_index=f))
    return intr, frames


def small_lr_config(**kw):
    cfg = api.default_config(lambda_trust=0.1, **kw)
    for f in ("lr_proj", "lr_dict", "lr_rotation", "lr_color", "lr_log_scale", "lr_opacity", "lr_feature"):
        setattr(cfg, f, 1e-4)
    cfg.lr_position = 1e-5
    return cfg


def pipeline_config(**kw):
    base = dict(query_dim=4, embed_dim=32, dict_size=16, stage1_iters=2, stage2_iters=2, history_sample=2,
                history_capacity=3, voxel_size=0.05, local_radius=3.0, sync_distance=0.5, hash_capacity=1 << 16,
                keyframe_stride=1, seed=7)
    base.update(kw)
    return api.default_pipeline_config(**base)


def f32_row_normalize(feats):
    """normalize_embedding_rows (pipeline.cpp:125-130): sequential float sum of squares."""
    out = feats.astype(np.float32).copy()
    for r in range(out.shape[0]):
        s = np.cumsum(out[r] * out[r], dtype=np.float32)[-1]
        n = np.float32(np.sqrt(s))
        if n > np.float32(1e-12):
            out[r] = out[r] / n
    return out


def composed_run(ctx, L, cfg, pc, intr, frames):
    """process_keyframe x len(frames) + the final flush, composed from pipeline.cpp:106-330."""
    qd, ed, K = pc.query_dim, pc.embed_dim, pc.dict_size
    rng = L.rng_new(pc.seed)
    s = api.Session(ctx, cfg, 0, qd, K, ed, intr)
    s.set_graphs(pc.stage1_iters >= 3)
    store = api.Store(ctx, pc.hash_capacity, qd)
    proj = np.zeros(qd * ed, np.float32)
    L.rng_normal(rng, 0.1, proj.size, proj.ctypes.data)
    s.set_dictionary(np.zeros((K, ed), np.float32), np.zeros((K, ed), np.float32), proj.reshape(qd, ed))
    s.set_dict_weights(np.zeros(K, np.float32))
    hist, head = [], 0
    origin, dirty = np.zeros(0, np.int64), np.zeros(0, np.uint8)
    traveled, last = np.float32(0), None
    logs = []

    def sync(center):
        nonlocal origin, dirty
        n = s.n
        rows = s.export_rows() if n else None
        d_out, org, kept, stats = store.sync(rows, origin, dirty, np.asarray(center, np.float32), pc.local_radius,
                                             pc.voxel_size)
        s.import_rows(d_out.contiguous(), kept=kept if n else None)
        origin, dirty = org, np.zeros(len(org), np.uint8)
        return stats

    for kf in frames:
        k = lamt.Keyframe(kf.pose_rot, kf.pose_trans, kf.rgb, kf.depth, kf.assignment, f32_row_normalize(kf.features),
                          frame_index=kf.frame_index)
        s.stream_kmeans(k.features, lambda: L.rng_uniform01(rng), decay=pc.dict_decay)
        idx = np.zeros(max(pc.history_sample, 1), np.int64)
        m = L.rng_sample_history(rng, len(hist), pc.history_sample, idx.ctypes.data)
        batch = [k] + [hist[i] for i in idx[:m]]
        s.set_frames(batch)
        rows = s.seed_candidates(0)
        nb = rows.shape[0]
        feats = np.zeros(nb * qd, np.float32)
        L.rng_normal(rng, 0.01, feats.size, feats.ctypes.data)
        if nb:
            s.append_rows(rows, feats.reshape(nb, qd))
        origin = np.concatenate([origin, -np.ones(nb, np.int64)])
        dirty = np.concatenate([dirty, np.ones(nb, np.uint8)])
        loss = None
        for _ in range(pc.stage1_iters):
            loss = s.step(read=True)
            dirty[:] = 1
        for _ in range(pc.stage2_iters):
            loss = s.step_dict(read=True)
        if len(hist) < pc.history_capacity:
            hist.append(k)
        else:
            hist[head] = k
            head = (head + 1) % pc.history_capacity
        t = np.asarray(k.pose_trans, np.float32)
        if last is not None:
            d = t - last
            traveled = np.float32(traveled + np.float32(np.sqrt(np.float32(np.float32(d[0] * d[0] + d[1] * d[1])
                                                                           + d[2] * d[2]))))
        last = t
        row = {"seeded": nb, "synced": False, "loss": loss}
        if traveled >= np.float32(pc.sync_distance):
            row["sync"] = sync(t)
            row["synced"] = True
            traveled = np.float32(0)
        row["active_count"], row["global_count"] = s.n, store.size()
        logs.append(row)
    flush = None
    if s.n:
        dirty[:] = 1
        flush = sync(last)
    return s, store, logs, flush, origin


def test_pipeline_matches_composed_loop(ctx, stdrng):
    intr, frames = make_scene(ctx)
    cfg, pc = small_lr_config(), pipeline_config()
    p = api.Pipeline(ctx, cfg, pc, intr)
    got = [p.process_keyframe(kf) for kf in frames]
    st = p.state()
    assert st["keyframes_processed"] == len(frames) and st["history"] == pc.history_capacity
    org_before_flush = p.active_set()[0]
    fl = p.flush()
    s2, store2, want, fl2, origin2 = composed_run(ctx, stdrng, cfg, pc, intr, frames)
    assert any(r["synced"] for r in got) and not all(r["synced"] for r in got)
    for a, b in zip(got, want):
        assert a["seeded"] == b["seeded"] and a["synced"] == b["synced"]
        assert a["active_count"] == b["active_count"] and a["global_count"] == b["global_count"]
        if a["synced"]:
            assert a["sync"] == b["sync"]
        for key in ("l_rgb", "l_depth", "l_cos", "l_l2", "total"):
            assert a["loss"][key] == pytest.approx(b["loss"][key], rel=2e-3, abs=1e-6), key
        assert a["loss"]["supervised_rows"] == b["loss"]["supervised_rows"]
    assert fl == fl2
    assert np.array_equal(p.active_set()[0], origin2) and len(org_before_flush) == got[-1]["active_count"]
    r1, k1 = p.store.records()
    r2, k2 = store2.records()
    assert np.array_equal(k1, k2)
    assert np.allclose(r1, r2, rtol=1e-3, atol=2e-3)
    a1, pr1 = p.session.get_dictionary()
    a2, pr2 = s2.get_dictionary()
    assert np.allclose(a1, a2, atol=2e-3) and np.allclose(pr1, pr2, atol=2e-3)
    assert np.array_equal(p.session.dict_weights(), s2.dict_weights())  # k-means masses are exact
    assert got[0]["dict_weight_mass"] == float(np.float32(frames[0].features.shape[0]))


def test_pipeline_random_dictionary_and_persistent_anchor(ctx):
    """dict_init = "random" (reservoir fills atoms in arrival order, anchor = atoms) and
    trust_anchor_persistent (the first keyframe's anchor is kept)."""
    intr, frames = make_scene(ctx, nframes=3, seed=1)
    pc = pipeline_config(dict_init="random", trust_anchor_persistent=1, stage1_iters=1, stage2_iters=0,
                         local_mapping=0)
    p = api.Pipeline(ctx, small_lr_config(), pc, intr)
    p.process_keyframe(frames[0])
    atoms0 = p.session.get_dictionary()[0].copy()
    anchor0 = p.session.get_anchor()
    nf = frames[0].features.shape[0]
    assert np.allclose(anchor0[:nf], f32_row_normalize(frames[0].features), atol=1e-6)
    assert (anchor0[nf:] == 0).all()
    w = p.session.dict_weights()
    assert (w[:nf] == 1).all() and (w[nf:] == 0).all()
    p.process_keyframe(frames[1])
    assert p.state()["reservoir_seen"] == 2 * nf
    assert np.array_equal(p.session.get_anchor(), anchor0)  # persistent
    assert not np.array_equal(p.session.get_dictionary()[0][nf:2 * nf], atoms0[nf:2 * nf])
    assert p.store.size() == 0  # local_mapping off: no sync


def test_pipeline_argument_errors_leave_state(ctx):
    intr, frames = make_scene(ctx, nframes=2, seed=2)
    p = api.Pipeline(ctx, small_lr_config(), pipeline_config(), intr)
    p.process_keyframe(frames[0])
    before = p.state()
    bad = lamt.Keyframe(frames[1].pose_rot, frames[1].pose_trans, frames[1].rgb, frames[1].depth,
                        np.full_like(frames[1].assignment, 6), frames[1].features)
    with pytest.raises(api._capi.InvalidArgument, match="assignment index out of range"):
        p.process_keyframe(bad)
    assert p.state() == before
    p.process_keyframe(frames[1])  # still usable
    with pytest.raises(api._capi.InvalidArgument, match="history sizes"):
        api.Pipeline(ctx, small_lr_config(), pipeline_config(history_capacity=0), intr)


def test_run_pipeline_over_lamt_dataset(ctx, tmp_path):
    """run_pipeline (pipeline.cpp:314-335): keyframe stride, LAMT frames, final flush into the
    store, CSV log rows."""
    intr, frames = make_scene(ctx, nframes=5, seed=3)
    li = lamt.Intrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height)
    lamt.save_dataset(str(tmp_path), li, frames)
    m = lamt.load_manifest(str(tmp_path))
    p = api.Pipeline(ctx, small_lr_config(), pipeline_config(keyframe_stride=2, local_mapping=0), intr)
    seen = []
    res = pl.run_pipeline(p, m, on_keyframe=seen.append)
    assert res["frames"] == 5 and res["keyframes"] == 3 and [r["frame_index"] for r in res["log"]] == [0, 2, 4]
    assert len(seen) == 3 and res["keyframes_per_second"] > 0
    assert p.store.size() > 0 and p.store.size() <= res["log"][-1]["active_count"]
    assert (p.active_set()[0] >= 0).all()  # every kept row now has a store record
    line = pl.log_csv_row(res["log"][0])
    assert len(line.split(",")) == len(pl.log_csv_header().split(","))


@pytest.mark.parametrize("stage", [1, 2, 3])
def test_process_keyframe_rolls_back_a_failed_keyframe(ctx, stage):
    """process_keyframe is a transaction (pipeline.cpp:292-306): a keyframe that fails after it
    started mutating the state (seeding appended rows, Stage I/II stepped the map, dictionary and
    moments, the sync re-homed the active set) leaves the ActiveSet rows / origin / dirty, the
    dictionary, the counters and the travel exactly as before it, and the pipeline continues; the
    repeated keyframe then matches a run that never failed. As in the reference the history
    buffer and the store are outside the snapshot (pipeline.cpp:155-169)."""
    intr, frames = make_scene(ctx, nframes=4)
    cfg, pc = small_lr_config(), pipeline_config()
    p = api.Pipeline(ctx, cfg, pc, intr)
    for kf in frames[:2]:
        p.process_keyframe(kf)

    def snapshot():
        s = p.session
        rows = s.export_rows().cpu().numpy().copy() if s.n else None
        atoms, proj = s.get_dictionary()
        st = p.state()
        st.pop("history")
        org, dty = p.active_set()
        return rows, atoms, proj, s.get_anchor(), s.dict_weights(), st, org, dty

    before = snapshot()
    p.inject_fault(stage)
    with pytest.raises(api._capi.LatmapError, match="injected fault"):
        p.process_keyframe(frames[2])
    after = snapshot()
    assert not p.state()["failed"]
    for a, b in zip(before, after):
        if isinstance(a, dict):
            assert a == b
        elif a is None:
            assert b is None
        else:
            assert np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))
    got = p.process_keyframe(frames[2])
    # a pipeline that never failed
    q = api.Pipeline(ctx, cfg, pc, intr)
    for kf in frames[:2]:
        q.process_keyframe(kf)
    ref = q.process_keyframe(frames[2])
    for k in ("seeded", "active_count", "synced"):
        assert got[k] == ref[k], k
    if stage != 3:  # a rolled-back sync already moved records into the store
        assert got["global_count"] == ref["global_count"]
    assert got["loss"]["total"] == pytest.approx(ref["loss"]["total"], rel=1e-3)


def test_pipeline_matches_reference_pipeline(ctx):
    """api.Pipeline against the REFERENCE's own pipeline (oracle/_ref: PipelineState,
    process_keyframe and run_pipeline's final flush compiled from proj/src/pipeline.cpp) on the
    same keyframes and configuration -- an independent check of csrc/pipeline.cu. Blend decisions
    are made bit-exact (exact blend mode) so seeding sees the reference's images; the Stage-I
    gradients differ from the reference's by float summation order only, and small learning
    rates keep that noise away from the seeding thresholds. Counts, sync statistics and active
    origins must match exactly; losses and the dictionary to float noise."""
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    intr, frames = make_scene(ctx)
    cfg, pc = small_lr_config(), pipeline_config()
    ctx.set_exact_blend(True)
    try:
        p = api.Pipeline(ctx, cfg, pc, intr)
        got = [p.process_keyframe(kf) for kf in frames]
        fl = p.flush()
    finally:
        ctx.set_exact_blend(False)
    rcfg = ref.make_config(num_threads=8, dict_learn=bool(cfg.dict_learn), segment_mode=bool(cfg.segment_mode),
                           **{f: getattr(cfg, f) for f in ref.CFG_FIELDS})
    rpc = ref.PipelineConfig(*[getattr(pc, f) for f, _ in ref.PipelineConfig._fields_])
    rp = ref.Pipeline(rcfg, rpc, intr)
    want = [rp.process_keyframe(kf) for kf in frames]
    rfl = rp.flush()
    assert any(r["synced"] for r in want) and any(r["seeded"] for r in want)
    for a, b in zip(got, want):
        assert (a["seeded"], a["synced"], a["active_count"], a["global_count"]) == (
            b["seeded"], b["synced"], b["active_count"], b["global_count"]), (a, b)
        if a["synced"]:
            assert a["sync"] == b["sync"]
        assert a["loss"]["supervised_rows"] == b["loss"]["supervised_rows"]
        for key in ("l_rgb", "l_depth", "l_cos", "l_l2", "total"):
            assert a["loss"][key] == pytest.approx(b["loss"][key], rel=2e-3, abs=1e-6), key
        assert a["dict_weight_mass"] == pytest.approx(b["dict_weight_mass"], rel=1e-5)
    assert fl == rfl
    rs = rp.state()
    assert np.array_equal(p.active_set()[0], rs["origin"])
    assert p.store.size() == rs["store_size"]
    atoms, proj = p.session.get_dictionary()
    np.testing.assert_allclose(atoms, rs["atoms"], rtol=1e-3, atol=1e-5)
    np.testing.assert_allclose(proj, rs["proj"], rtol=1e-3, atol=1e-5)
