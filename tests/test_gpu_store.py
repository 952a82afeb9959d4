"""Device voxel-hash store (K11) against the oracle store: record indices, rejections, keys,
fetch_local lists and sync outputs must be bit-exact (BASELINE: hash lookups bit-exact)."""
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


def recs(rng, n, extent=2.0, ds=4):
    r = np.zeros((n, 14 + ds), np.float32)
    r[:, 0:3] = rng.uniform(-extent, extent, (n, 3))
    q = rng.standard_normal((n, 4))
    r[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    r[:, 7:] = rng.standard_normal((n, 7 + ds))
    return r


def test_insert_find_records_match(ctx):
    rng = np.random.default_rng(1)
    r = recs(rng, 20000)
    r[5000:6000, :3] = r[:1000, :3] + 1e-4  # duplicate voxels
    for cap in (1 << 16, 20011):
        s, o = api.Store(ctx, cap, 4), oracle.Store(cap, 4)
        assert s.insert_global(r, 0.01) == o.insert_global(r, 0.01)
        assert s.size() == o.size()
        assert s.stats() == o.stats()
        got, keys = s.records()
        assert np.array_equal(got.view(np.uint32), o.records().view(np.uint32))
        assert all(tuple(keys[i]) == o.record_key(i) for i in range(0, s.size(), 97))
        for p in r[::53, :3]:
            k = oracle.voxel_of(p, 0.01)
            assert s.find(k) == o.find(k)


def test_overflow_chain(ctx):  # test_store.cpp:106-124
    cap = 64
    target = oracle.hash_voxel((0, 0, 0), cap)
    chain, ix = [], 0
    while len(chain) <= 8:
        if oracle.hash_voxel((ix, 0, 0), cap) == target:
            chain.append((ix, 0, 0))
        ix += 1
    s = api.Store(ctx, cap, 4)
    rec = np.zeros(18, np.float32)
    for k in chain[:-1]:
        assert s.insert(k, rec) >= 0
    assert s.insert(chain[-1], rec) == -1
    assert s.stats()["rejected_overflow"] == 1


def test_fetch_local_matches(ctx):
    rng = np.random.default_rng(2)
    r = recs(rng, 30000)
    s, o = api.Store(ctx, 1 << 17, 4), oracle.Store(1 << 17, 4)
    s.insert_global(r, 0.01)
    o.insert_global(r, 0.01)
    pool = o.records()
    for t in range(60):
        c = rng.uniform(-2, 2, 3).astype(np.float32)
        rad = np.float32(rng.uniform(0.05, 2.5))
        idx, d = s.fetch_local(c, rad, gather=True)
        ref = o.fetch_local(c, rad)
        assert np.array_equal(idx, ref)
        assert np.array_equal(d.cpu().numpy().view(np.uint32), pool[ref].view(np.uint32))
    assert len(s.fetch_local((0, 0, 0), 1e-3)) >= 0
    with pytest.raises(ValueError):
        s.fetch_local((0, 0, 0), 0.0)


def test_sync_sequence_matches(ctx):
    rng = np.random.default_rng(3)
    s, o = api.Store(ctx, 1 << 16, 4), oracle.Store(1 << 16, 4)
    base = recs(rng, 3000)
    s.insert_global(base, 0.05)
    o.insert_global(base, 0.05)
    center = np.zeros(3, np.float32)
    org = o.fetch_local(center, 1.0)
    act = o.records()[org]
    dirty = np.zeros(len(org), np.uint8)
    for step in range(6):
        # optimisation moves some tracked entries (possibly across voxels), adds newborns
        act = act.copy()
        moved = rng.random(len(act)) < 0.3
        act[moved, :3] += rng.normal(0, 0.05, (moved.sum(), 3)).astype(np.float32)
        act[moved, 7:] += 0.1
        dirty = moved.astype(np.uint8)
        born = recs(rng, 50, extent=1.5)
        born[:10, :3] = act[:10, :3]  # some land in occupied voxels -> rejected
        act = np.concatenate([act, born])
        org = np.concatenate([org, -np.ones(50, np.int64)])
        dirty = np.concatenate([dirty, np.ones(50, np.uint8)])
        center = (center + rng.normal(0, 0.3, 3)).astype(np.float32)
        d_out, g_org, g_kept, g_st = s.sync(torch.as_tensor(act, device="cuda"), org, dirty, center, 1.0, 0.05)
        r_out, r_org, r_kept, r_st = o.sync(act, org, dirty, center, 1.0, 0.05)
        assert g_st == r_st, (step, g_st, r_st)
        assert np.array_equal(g_org, r_org) and np.array_equal(g_kept, r_kept)
        assert np.array_equal(d_out.cpu().numpy().view(np.uint32), r_out.view(np.uint32))
        assert np.array_equal(s.records()[0].view(np.uint32), o.records().view(np.uint32))
        act, org = r_out, r_org


def test_streaming_session_loop_matches_oracle_store(ctx):
    """Config-3 loop at reduced scale: per frame store sync of the session's optimised active
    set -> row import -> Stage-I steps. The active set (row order, origins, kept masks) must match
    the oracle store's sync run on the same rows bit for bit, and the steps must stay finite.
    An odd active count exercises the session's block alignment."""
    from paper_2602_12314_b200 import synthetic

    st = synthetic.make_streaming(n_global=1_000_000, nframes=3, scale=0.2, device="cuda")  # 40k records
    intr = api.make_intrinsics(st.intr.fx, st.intr.fy, st.intr.cx, st.intr.cy, st.intr.width, st.intr.height)
    store = api.Store(ctx, st.capacity, 32)
    ostore = oracle.Store(st.capacity, 32)
    store.insert_global(st.records, st.voxel_size)
    ostore.insert_global(st.records, st.voxel_size)
    cfg = api.default_config(**st.lambdas)
    cfg.decoder_precision = 1
    s = api.Session(ctx, cfg, 0, 32, 256, 1024, intr)
    s.set_dictionary(st.atoms, st.atoms, st.proj)
    origin = np.zeros(0, np.int64)
    ncount = []
    for f, (q, t) in enumerate(st.poses):
        rows = s.export_rows() if s.n else None
        host_rows = rows.cpu().numpy() if rows is not None else np.zeros((0, 46), np.float32)
        dirty = np.ones(len(origin), np.uint8)
        d_out, org, kept, stats = store.sync(rows, origin, dirty, np.asarray(t, np.float32), st.radius, st.voxel_size)
        o_out, o_org, o_kept, o_stats = ostore.sync(host_rows, origin, dirty, np.asarray(t, np.float32), st.radius,
                                                     st.voxel_size)
        assert np.array_equal(org, o_org) and np.array_equal(kept, np.asarray(o_kept, bool))
        assert np.array_equal(d_out.cpu().numpy(), o_out)
        s.import_rows(d_out.contiguous(), kept=kept if len(origin) else None)
        origin = org
        ncount.append(s.n)
        h, w = st.intr.height, st.intr.width
        rgb = np.full((h, w, 3), 0.5, np.float32)
        dep = np.full((h, w), 3.0, np.float32)
        s.set_frames([synthetic.Frame(q, t, rgb, dep, st.assignments[f], st.features[f])])
        s.set_batch(1)
        for _ in range(2):
            loss = s.step(read=True)
        assert np.isfinite(loss["total"])
    assert min(ncount) > 0


def test_map_dump_restore_round_trip(ctx, tmp_path):
    """save_map_store -> load_map_store -> a fresh store rebuilt under the dumped keys
    (artifacts.cpp:40-63): same records in the same order, same keys, same find() answers,
    and fetch_local over the rebuilt store equals the original's."""
    from paper_2602_12314_b200 import lamt
    rng = np.random.default_rng(11)
    r = recs(rng, 5000)
    s = api.Store(ctx, 1 << 15, 4)
    s.insert_global(r, 0.01)
    lamt.save_map_store(s, str(tmp_path / "map.lamt"))
    lamt.save_store_counters(s, str(tmp_path / "counters.json"))
    lm = lamt.load_map_store(str(tmp_path / "map.lamt"))
    t = lamt.restore_store(ctx, lm, 1 << 15)
    assert t.size() == s.size()
    a, ka = s.records()
    b, kb = t.records()
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32)) and np.array_equal(ka, kb)
    for k in ka[::41]:
        assert t.find(k) == s.find(k)
    c = np.array([0.3, -0.2, 0.1], np.float32)
    assert np.array_equal(t.fetch_local(c, 1.0), s.fetch_local(c, 1.0))
    # a different capacity changes the slots, not the record order
    u = lamt.restore_store(ctx, lm, 20011)
    assert np.array_equal(u.records()[0].view(np.uint32), a.view(np.uint32))
    assert u.insert_keyed(ka[:3], a[:3]) == 0 and u.stats()["rejected_duplicate"] == 3


def test_session_dictionary_dump_round_trip(ctx, tmp_path):
    """save_dictionary of a device session -> load_dictionary -> apply to another session."""
    from paper_2602_12314_b200 import lamt
    g = np.random.default_rng(12)
    k, df, ds = 16, 32, 8
    cfg = api.default_config(softmax_temp=2.0)
    intr = api.make_intrinsics(50, 50, 16, 16, 32, 32)
    s1, s2 = (api.Session(ctx, cfg, 16, ds, k, df, intr) for _ in range(2))
    atoms, anchor = g.standard_normal((2, k, df)).astype(np.float32)
    proj = g.standard_normal((ds, df)).astype(np.float32)
    s1.set_dictionary(atoms, anchor, proj)
    s1.set_dict_weights(g.uniform(0, 4, k).astype(np.float32))
    lamt.save_dictionary(s1, str(tmp_path / "dict.lamt"))
    d = lamt.load_dictionary(str(tmp_path / "dict.lamt"))
    assert d.temperature == 2.0 and np.array_equal(d.anchor, anchor)
    lamt.apply_dictionary(s2, d)
    a2, p2 = s2.get_dictionary()
    assert np.array_equal(a2, atoms) and np.array_equal(p2, proj)
    assert np.array_equal(s2.get_anchor(), anchor) and np.array_equal(s2.dict_weights(), s1.dict_weights())


def test_sync_device_matches_host_sync(ctx):
    """latmap_store_sync_device (per-row arrays on the device, device compactions) against the host
    sync on the same sequence: outputs, origins, kept masks, stats and the stored records bit for
    bit, with newborns (some rejected), tracked moves across voxels and a drifting centre; one
    frame with every row dirty (d_dirty = None)."""
    rng = np.random.default_rng(5)
    a, b = api.Store(ctx, 1 << 16, 4), api.Store(ctx, 1 << 16, 4)
    base = recs(rng, 4000)
    a.insert_global(base, 0.05)
    b.insert_global(base, 0.05)
    center = np.zeros(3, np.float32)
    org, act_t = a.fetch_local(center, 1.0, gather=True)
    b.fetch_local(center, 1.0)
    act = act_t.cpu().numpy()
    for step in range(6):
        act = act.copy()
        moved = rng.random(len(act)) < 0.3
        act[moved, :3] += rng.normal(0, 0.05, (moved.sum(), 3)).astype(np.float32)
        act[moved, 7:] += 0.1
        dirty = moved.astype(np.uint8)
        nb = 0 if step == 2 else 60
        if nb:
            born = recs(rng, nb, extent=1.5)
            born[:10, :3] = act[:10, :3]
            act = np.concatenate([act, born])
            org = np.concatenate([org, -np.ones(nb, np.int64)])
            dirty = np.concatenate([dirty, np.ones(nb, np.uint8)])
        all_dirty = step == 4
        if all_dirty:
            dirty = np.ones(len(org), np.uint8)
        center = (center + rng.normal(0, 0.3, 3)).astype(np.float32)
        d_act = torch.as_tensor(act, device="cuda")
        h_out, h_org, h_kept, h_st = a.sync(d_act, org, dirty, center, 1.0, 0.05)
        d_out, d_org, d_kept, d_st = b.sync_device(d_act, torch.as_tensor(org, device="cuda"),
                                                   None if all_dirty else torch.as_tensor(dirty, device="cuda"),
                                                   center, 1.0, 0.05)
        assert d_st == h_st, (step, d_st, h_st)
        assert np.array_equal(d_org.cpu().numpy(), h_org)
        assert np.array_equal(d_kept.cpu().numpy().astype(bool), h_kept)
        assert np.array_equal(d_out.cpu().numpy().view(np.uint32), h_out.cpu().numpy().view(np.uint32))
        assert a.size() == b.size()
        assert np.array_equal(a.records()[0].view(np.uint32), b.records()[0].view(np.uint32))
        act, org = h_out.cpu().numpy(), h_org


def test_import_rows_device_matches_host(ctx):
    """Session.import_rows_device (kept mask on the device) == import_rows (host mask): in
    deterministic mode, one Stage-I step, the row import, and a second step (whose Adam update
    depends on the carried moments) give bit-identical maps. Also: deterministic mode switched on
    after a graph-captured step (its scratch must be sized outside the re-capture)."""
    from paper_2602_12314_b200 import synthetic

    st = synthetic.make_streaming(n_global=1_000_000, nframes=1, scale=0.1, device="cuda")
    intr = api.make_intrinsics(st.intr.fx, st.intr.fy, st.intr.cx, st.intr.cy, st.intr.width, st.intr.height)
    store = api.Store(ctx, st.capacity, 32)
    store.insert_global(st.records, st.voxel_size)
    q, t = st.poses[0]
    org, rows = store.fetch_local(np.asarray(t, np.float32), st.radius, gather=True)
    gm = api.GaussianMap(rows[:, 0:3].contiguous(), rows[:, 3:7].contiguous(), rows[:, 7:10].contiguous(),
                         rows[:, 10:13].contiguous(), rows[:, 13].contiguous(), rows[:, 14:].contiguous())
    out = api.render(ctx, gm, api.make_pose(q, t), intr)
    frame = synthetic.Frame(q, t, out.color.cpu().numpy() * 0.9, out.depth.cpu().numpy(), st.assignments[0],
                            st.features[0])
    cfg = api.default_config(**st.lambdas)
    rng = np.random.default_rng(1)
    kept = rng.random(len(org)) < 0.7
    new_rows = torch.cat([rows[torch.as_tensor(kept, device="cuda")], rows[:100]]).contiguous()
    res = []
    for dev in (False, True):
        s = api.Session(ctx, cfg, 0, 32, 256, 1024, intr)
        s.set_dictionary(st.atoms, st.atoms, st.proj)
        s.import_rows(rows.contiguous())
        s.set_frames([frame])
        s.set_batch(1)
        ctx.set_deterministic(True)
        try:
            s.step(read=True)
            s.step(read=True)  # graph-captured
            if dev:
                s.import_rows_device(new_rows, torch.as_tensor(kept, device="cuda"), int(kept.sum()))
            else:
                s.import_rows(new_rows, kept=kept)
            s.step(read=True)
            s.step(read=True)
        finally:
            ctx.set_deterministic(False)
        res.append(s.params_buffer().clone())
        del s
    assert torch.equal(res[0], res[1])
    # deterministic mode switched on after a graph-captured step: the fixed-order scratch is sized
    # before the re-capture (an allocation inside a capture fails)
    s = api.Session(ctx, cfg, 0, 32, 256, 1024, intr)
    s.set_dictionary(st.atoms, st.atoms, st.proj)
    s.import_rows(rows.contiguous())
    s.set_frames([frame])
    s.set_batch(1)
    s.step(read=True)
    s.step(read=True)
    ctx.set_deterministic(True)
    try:
        assert np.isfinite(s.step(read=True)["total"])
    finally:
        ctx.set_deterministic(False)


def test_fetch_local_device_matches_host(ctx):
    """fetch_local_device (single-pass look-back compaction) == fetch_local: the ascending record
    list and the gathered records, over a 300k-record store at several radii (block boundaries,
    empty and full results)."""
    rng = np.random.default_rng(9)
    s = api.Store(ctx, 1 << 20, 4)
    s.insert_global(recs(rng, 300_000, extent=4.0), 0.01)
    for radius in (0.05, 0.7, 2.0, 100.0):
        c = rng.normal(0, 1, 3).astype(np.float32)
        h_org, h_rec = s.fetch_local(c, radius, gather=True)
        d_org, d_rec = s.fetch_local_device(c, radius, gather=True)
        assert np.array_equal(d_org.cpu().numpy(), h_org), radius
        assert torch.equal(d_rec, h_rec), radius
