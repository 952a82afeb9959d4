"""Pins the CPU oracle's objective, Adam and voxel-hash store against the
reference's own suites (proj/tests/test_objective.cpp, proj/tests/test_store.cpp)."""
import math

import numpy as np
import pytest

import oracle
from tests.helpers import grad_check, random_map, small_intrinsics


def objective_config():  # test_objective.cpp:79-85 (defaults of config.hpp)
    return oracle.Config()


def random_dict(k, ds, df, rng):  # test_objective.cpp:68-77
    atoms = rng.standard_normal((k, df)) * 0.5
    return oracle.Dictionary(atoms, atoms.copy(), rng.standard_normal((ds, df)) * 0.5, 1.0)


def self_consistent_frame(m, d, intr):  # test_objective.cpp:17-44
    out = oracle.render(m, (1, 0, 0, 0), (0, 0, 0), intr)
    h, w = intr.height, intr.width
    depth = np.where(out["alpha"] > 0.5, out["depth"], 0.0)
    assign = np.arange(h * w, dtype=np.int32)
    feats = oracle.reconstruct(out["query"].reshape(h * w, -1), d.atoms, d.proj, d.temperature)
    return oracle.Frame((1, 0, 0, 0), (0, 0, 0), out["color"], depth, assign, feats)


def random_frame(intr, df, rng):  # test_objective.cpp:46-66
    h, w = intr.height, intr.width
    feats = rng.standard_normal((h * w, df))
    feats /= np.linalg.norm(feats, axis=1, keepdims=True)
    return oracle.Frame((1, 0, 0, 0), (0, 0, 0), rng.random((h, w, 3)), 1 + 2 * rng.random((h, w)),
                        np.arange(h * w, dtype=np.int32), feats)


def test_fixed_point_scores_zero():  # test_objective.cpp:89-104
    rng = np.random.default_rng(21)
    intr = small_intrinsics(16, 16, 18.0)
    m = random_map(15, 4, rng)
    d = random_dict(8, 4, 12, rng)
    fr = self_consistent_frame(m, d, intr)
    loss, _ = oracle.total_objective(m, d, [fr], intr, objective_config(), want_grad=False)
    assert loss["total"] < 1e-3
    assert loss["l_rgb"] < 1e-9 and loss["l_depth"] < 1e-9 and loss["l_cos"] < 1e-9
    assert loss["l_trust"] == 0.0


def test_lambda_feat_zero_reduction():  # test_objective.cpp:106-120
    rng = np.random.default_rng(22)
    intr = small_intrinsics(12, 12, 14.0)
    m = random_map(8, 4, rng)
    d = random_dict(6, 4, 12, rng)
    fr = random_frame(intr, 12, rng)
    cfg = objective_config()
    cfg.lambda_feat = 0
    a, _ = oracle.total_objective(m, d, [fr], intr, cfg, want_grad=False)
    f = lambda x: float(np.float32(x))  # noqa: E731  (Config fields are float)
    expect = f(cfg.lambda_rgb) * (f(cfg.lambda_i1) * a["l_rgb"] + f(cfg.lambda_i2) * a["l_ssim"]) + \
        f(cfg.lambda_depth) * a["l_depth"]
    assert a["total"] == pytest.approx(expect, rel=1e-12)


def test_objective_nonnegative():  # test_objective.cpp:122-135
    rng = np.random.default_rng(23)
    intr = small_intrinsics(12, 12, 14.0)
    for _ in range(5):
        m = random_map(6, 4, rng)
        d = random_dict(5, 4, 12, rng)
        fr = random_frame(intr, 12, rng)
        loss, _ = oracle.total_objective(m, d, [fr], intr, objective_config(), want_grad=False)
        assert loss["total"] >= 0.0


def test_full_objective_fd():  # test_objective.cpp:137-170
    rng = np.random.default_rng(2025)
    intr = small_intrinsics(16, 16, 16.0)
    m = random_map(10, 4, rng)
    d = random_dict(8, 4, 12, rng)
    d.atoms = d.anchor + 0.05
    fr = random_frame(intr, 12, rng)
    cfg = objective_config()
    _, (g, dp, da) = oracle.total_objective(m, d, [fr], intr, cfg)
    loss = lambda: float(oracle.total_objective(m, d, [fr], intr, cfg, want_grad=False)[0]["total"])  # noqa
    assert grad_check(loss, m.positions, g.positions, max_coords=15) < 1e-3
    assert grad_check(loss, m.rotations, g.rotations, max_coords=15) < 1e-3
    assert grad_check(loss, m.colors, g.colors, max_coords=15) < 1e-3
    assert grad_check(loss, m.log_scales, g.log_scales, max_coords=15) < 1e-3
    assert grad_check(loss, m.opacity_logits, g.opacity_logits, max_coords=10) < 1e-3
    assert grad_check(loss, m.features, g.features, max_coords=15) < 1e-3
    assert grad_check(loss, d.proj, dp, max_coords=20) < 1e-3
    assert grad_check(loss, d.atoms, da, max_coords=30) < 1e-3


def test_multi_frame_batch_mean_fd():  # objective.cpp:77 (inv_b) with a 2-frame batch
    rng = np.random.default_rng(77)
    intr = small_intrinsics(12, 12, 14.0)
    m = random_map(8, 4, rng)
    d = random_dict(6, 4, 12, rng)
    d.atoms = d.anchor + 0.05
    frames = [random_frame(intr, 12, rng), random_frame(intr, 12, rng)]
    frames[1].pose_trans = (0.05, 0.0, 0.0)
    cfg = objective_config()
    _, (g, dp, da) = oracle.total_objective(m, d, frames, intr, cfg)
    loss = lambda: float(oracle.total_objective(m, d, frames, intr, cfg, want_grad=False)[0]["total"])  # noqa
    assert grad_check(loss, m.positions, g.positions, max_coords=12) < 1e-3
    assert grad_check(loss, m.features, g.features, max_coords=12) < 1e-3
    assert grad_check(loss, d.atoms, da, max_coords=12) < 1e-3


def test_segment_mode_fd():  # objective.cpp:37-64,147-157 (segment supervision)
    rng = np.random.default_rng(78)
    intr = small_intrinsics(12, 12, 14.0)
    m = random_map(8, 4, rng)
    d = random_dict(6, 4, 12, rng)
    d.atoms = d.anchor + 0.05
    fr = random_frame(intr, 12, rng)
    fr.assignment = (np.arange(144, dtype=np.int32) % 5)
    fr.assignment[::7] = -1
    fr.features = fr.features[:5].copy()
    cfg = objective_config()
    cfg.segment_mode = True
    _, (g, dp, da) = oracle.total_objective(m, d, [fr], intr, cfg)
    loss = lambda: float(oracle.total_objective(m, d, [fr], intr, cfg, want_grad=False)[0]["total"])  # noqa
    assert grad_check(loss, m.features, g.features, max_coords=12) < 1e-3
    assert grad_check(loss, d.proj, dp, max_coords=12) < 1e-3


def test_adam_zero_gradient():  # test_objective.cpp:181-187
    p = np.ones((3, 3), np.float32)
    st = oracle.AdamState(np.zeros_like(p), np.zeros_like(p))
    oracle.adam_step(p, np.zeros((3, 3), np.float32), st, 0.1)
    assert np.abs(p - 1).max() == 0


def test_adam_first_step_is_lr_sign():  # test_objective.cpp:189-200
    p = np.zeros((2, 2))
    g = np.array([[3.0, -0.2], [1e-3, -40.0]])
    st = oracle.AdamState(np.zeros_like(p), np.zeros_like(p))
    oracle.adam_step(p, g, st, 0.01)
    assert np.all(np.abs(np.abs(p) - 0.01) < 1e-5)
    assert p[0, 0] < 0 and p[1, 1] > 0


def test_adam_skips_nonfinite():  # test_objective.cpp:202-210
    p = np.ones((2, 2), np.float32)
    g = np.ones((2, 2), np.float32)
    g[1, 1] = np.nan
    st = oracle.AdamState(np.zeros_like(p), np.zeros_like(p))
    assert not oracle.adam_step(p, g, st, 0.1)
    assert st.skipped == 1 and np.abs(p - 1).max() == 0


def test_adam_quadratic_bowl():  # test_objective.cpp:212-222
    x = np.array([1.0, -0.75, 0.5])
    st = oracle.AdamState(np.zeros_like(x), np.zeros_like(x))
    for _ in range(500):
        oracle.adam_step(x, 2 * x, st, 0.01)
    assert np.abs(x).max() < 0.05


def test_trust_weight_keeps_atoms_near_ball():  # test_objective.cpp:224-244
    delta, lr, lt = 0.1, 1e-3, 1e5
    anchor = np.zeros((4, 6))
    atoms = anchor.copy()
    target = np.ones((4, 6))
    st = oracle.AdamState(np.zeros_like(atoms), np.zeros_like(atoms))
    worst = 0
    for _ in range(100):
        _, tg = oracle.trust_region_penalty(atoms, anchor, delta, want_grad=True)
        oracle.adam_step(atoms, 2 * (atoms - target) + lt * tg, st, lr)
        worst = max(worst, np.linalg.norm(atoms - anchor, axis=1).max())
    assert worst <= delta + 5 * lr and worst > 0.5 * delta


def test_one_step_from_anchor_stays_inside():  # test_objective.cpp:246-260
    rng = np.random.default_rng(31)
    anchor = rng.standard_normal((5, 8))
    atoms = anchor.copy()
    g = rng.standard_normal((5, 8))
    _, tg = oracle.trust_region_penalty(atoms, anchor, 0.1, want_grad=True)
    assert np.abs(tg).max() == 0
    st = oracle.AdamState(np.zeros_like(atoms), np.zeros_like(atoms))
    oracle.adam_step(atoms, g + 1e6 * tg, st, 0.01)
    assert np.all(np.linalg.norm(atoms - anchor, axis=1) <= 0.1)


def test_objective_decreases():  # test_objective.cpp:262-303
    intr = small_intrinsics(12, 12, 14.0)
    cfg = objective_config()
    improved = 0
    for t in range(10):
        rng = np.random.default_rng(1000 + t)
        m = random_map(8, 4, rng)
        d = random_dict(6, 4, 12, rng)
        fr = random_frame(intr, 12, rng)
        opt = oracle.MapOptimizer()
        first = None
        c2 = oracle.Config(lr_position=1e-4, lr_rotation=1e-3, lr_color=2.5e-3, lr_log_scale=5e-3,
                           lr_opacity=5e-2, lr_feature=2.5e-3, lr_proj=0.01, lr_dict=0.01)
        for it in range(20):
            loss, (g, dp, da) = oracle.total_objective(m, d, [fr], intr, cfg)
            if it == 0:
                first = loss["total"]
            opt.step_map(m, g, c2)
            opt.step_dict(d, dp, da, c2)
        last = oracle.total_objective(m, d, [fr], intr, cfg, want_grad=False)[0]["total"]
        improved += last < first
    assert improved >= 9


# ---------------------------------------------------------------------------- store
def prim(p, ds=4, tag=0.0):  # test_store.cpp:13-24
    return np.array(list(p) + [1, 0, 0, 0, tag, 0.5, 0.5, -3, -3, -3, 0.4] + [tag] * ds, np.float32)


def random_positions(n, rng, extent=2.0, ds=4):  # test_store.cpp:26-38
    r = np.zeros((n, 14 + ds), np.float32)
    r[:, 0:3] = rng.uniform(-extent, extent, (n, 3))
    r[:, 3] = 1
    r[:, 7:10] = rng.uniform(-extent, extent, (n, 1))
    r[:, 10:13] = -3
    r[:, 13] = rng.uniform(-extent, extent, n)
    r[:, 14:] = rng.uniform(-extent, extent, (n, 1))
    return r


def test_voxel_of():  # test_store.cpp:42-54
    assert oracle.voxel_of((0.015, -0.003, 0.021), 0.01) == (1, -1, 2)
    assert oracle.voxel_of((0, 0, 0), 0.01) == (0, 0, 0)
    assert oracle.voxel_of((0.01, 0.01, 0.01), 0.01) == (1, 1, 1)


def test_hash_known_values():  # test_store.cpp:56-64
    assert oracle.hash_voxel((0, 0, 0), 1 << 20) == 0
    assert oracle.hash_voxel((1, 0, 0), 1 << 20) == 73856093 % (1 << 20) == 455773
    for i in range(-5, 0):
        assert oracle.hash_voxel((i, 2 * i, -7 * i), 4096) >= 0


def test_hash_distribution():  # test_store.cpp:66-78
    rng = np.random.default_rng(17)
    cap = 1 << 17
    keys = rng.integers(-500, 501, (100000, 3))
    load = np.zeros(cap, np.int64)
    for k in keys:
        load[oracle.hash_voxel(tuple(int(v) for v in k), cap)] += 1
    assert load.max() <= 8


def test_insert_duplicate_rejection():  # test_store.cpp:80-94
    s = oracle.Store(4096, 4)
    assert s.insert(oracle.voxel_of((0.1, 0.2, 0.3), 0.01), prim((0.1, 0.2, 0.3))) >= 0
    assert s.size() == 1 and s.stats()["inserted"] == 1
    before = s.record(0)
    assert s.insert(oracle.voxel_of((0.101, 0.201, 0.301), 0.01), prim((0.101, 0.201, 0.301), 4, 9.0)) == -1
    assert s.size() == 1 and s.stats()["rejected_duplicate"] == 1
    assert s.record(0)[7] == before[7]


def test_update_in_place():  # test_store.cpp:96-104
    s = oracle.Store(4096, 4)
    key = oracle.voxel_of((0.1, 0.2, 0.3), 0.01)
    s.insert(key, prim((0.1, 0.2, 0.3)))
    assert s.update(key, prim((0.105, 0.2, 0.3), 4, 3.0))
    assert s.size() == 1 and s.record(0)[7] == 3.0
    assert not s.update((99, 99, 99), prim((1, 1, 1)))


def test_probe_chain_overflow():  # test_store.cpp:106-124
    cap = 64
    target = oracle.hash_voxel((0, 0, 0), cap)
    chain = []
    ix = 0
    while len(chain) <= 8:
        if oracle.hash_voxel((ix, 0, 0), cap) == target:
            chain.append((ix, 0, 0))
        ix += 1
    s = oracle.Store(cap, 4)
    for i, k in enumerate(chain[:-1]):
        assert s.insert(k, prim((i, 0, 0))) >= 0
    assert s.insert(chain[-1], prim((9, 9, 9))) == -1
    assert s.stats()["rejected_overflow"] == 1 and s.check_unique_keys()


def test_fetch_local_boundary():  # test_store.cpp:126-133
    s = oracle.Store(4096, 4)
    assert len(s.fetch_local((0, 0, 0), 1.0)) == 0
    s.insert(oracle.voxel_of((1.0, 0, 0), 0.01), prim((1.0, 0, 0)))
    assert len(s.fetch_local((0, 0, 0), 0.999)) == 0
    assert len(s.fetch_local((0, 0, 0), 1.001)) == 1


def test_fetch_local_linear_scan_oracle():  # test_store.cpp:159-184
    rng = np.random.default_rng(29)
    s = oracle.Store(1 << 16, 4)
    s.insert_global(random_positions(1000, rng), 0.01)
    pool = s.records()
    for _ in range(200):
        c = rng.uniform(-2, 2, 3).astype(np.float32)
        r = np.float32(rng.uniform(0.1, 2.5))
        got = s.fetch_local(c, r)
        d = pool[:, :3] - c
        expect = np.nonzero((d * d).sum(1) <= r * r)[0]
        assert np.array_equal(got, expect)


def test_sync_idempotent():  # test_store.cpp:186-203
    rng = np.random.default_rng(31)
    s = oracle.Store(1 << 16, 4)
    s.insert_global(random_positions(300, rng), 0.01)
    org = s.fetch_local((0, 0, 0), 1.5)
    recs = s.records()[org]
    b, bo, _, s1 = s.sync(recs, org, np.zeros(len(org), np.uint8), (0, 0, 0), 1.5, 0.01)
    c, co, _, s2 = s.sync(b, bo, np.zeros(len(bo), np.uint8), (0, 0, 0), 1.5, 0.01)
    assert s1["written_back"] == 0 and len(b) == len(org) and len(c) == len(b) and s2["fetched"] == 0
    assert np.array_equal(bo, co) and np.array_equal(b[:, :3], c[:, :3])


def test_sync_newborn_outside_radius():  # test_store.cpp:205-220
    s = oracle.Store(4096, 4)
    born = prim((5, 0, 0))[None]
    nxt, no, _, st = s.sync(born, np.array([-1]), np.array([1], np.uint8), (0, 0, 0), 2.0, 0.01)
    assert st["newborn_inserted"] == 1 and s.size() == 1 and len(nxt) == 0


def test_sync_drift_keeps_origin():  # test_store.cpp:222-241
    s = oracle.Store(4096, 4)
    p0 = (0.0501, 0.02, 0.02)
    s.insert(oracle.voxel_of(p0, 0.1), prim(p0))
    org = s.fetch_local((0, 0, 0), 1.0)
    recs = s.records()[org]
    recs[0, 0] = -0.01
    nxt, no, _, st = s.sync(recs, org, np.array([1], np.uint8), (0, 0, 0), 1.0, 0.1)
    assert st["written_back"] == 1 and s.size() == 1
    assert s.records()[0, 0] == np.float32(-0.01)
    assert s.record_key(0) == oracle.voxel_of(p0, 0.1)
    assert len(nxt) == 1 and no[0] == 0


def test_unique_keys_after_random_ops():  # test_store.cpp:243-264
    rng = np.random.default_rng(37)
    s = oracle.Store(2048, 4)
    pts = rng.uniform(-1, 1, (20000, 3)).astype(np.float32)
    for op, p in enumerate(pts):
        k = oracle.voxel_of(p, 0.05)
        if op % 4 in (0, 1):
            s.insert(k, prim(p))
        elif op % 4 == 2:
            s.update(k, prim(p, 4, 1.0))
        else:
            s.find(k)
    assert s.check_unique_keys() and s.size() <= 2048
