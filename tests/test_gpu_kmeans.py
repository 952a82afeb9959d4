"""Streaming k-means dictionary maintenance on the GPU against the oracle
restatement of proj/src/stream_kmeans.cpp, bit for bit: both sides draw k-means++ picks from
identically seeded std::mt19937_64 generators (oracle.MT64), so centres, masses, iteration counts
and the maintained dictionary must agree exactly."""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2602_12314_b200 import _capi, api  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return api.Context(0)


def gen(rng):
    """(C function pointer, user pointer) drawing uniform01 from an oracle MT64 state."""
    return oracle.MT64.uniform01_fn(), C.cast(C.byref(rng), C.c_void_p).value


def clustered(seed, n, dim, centres=6, spread=0.3):
    g = np.random.default_rng(seed)
    mu = g.standard_normal((centres, dim)) * 3
    lab = g.integers(0, centres, n)
    return (mu[lab] + spread * g.standard_normal((n, dim))).astype(np.float32)


@pytest.mark.parametrize("n,dim,k,n_warm,zero_w", [
    (200, 64, 16, 0, False),    # k-means++ from scratch
    (300, 48, 24, 10, False),   # warm start + 14 draws
    (120, 32, 8, 0, True),      # some zero weights
    (40, 16, 64, 0, False),     # k > n: exhausted mass, wrap-around picks, zero-weight duplicates
    (90, 40, 12, 12, False),    # fully warm (no draws)
])
def test_weighted_kmeans_bit_exact(ctx, n, dim, k, n_warm, zero_w):
    pts = clustered(n * 7 + dim, n, dim)
    w = np.random.default_rng(n).uniform(0.5, 2.0, n).astype(np.float32)
    if zero_w:
        w[::5] = 0
    warm = pts[:n_warm] + 0.05 if n_warm else None
    r_gpu, r_cpu = oracle.MT64(1000 + n), oracle.MT64(1000 + n)
    cg, wg, ig = ctx.weighted_kmeans(pts, w, k, gen(r_gpu), warm=warm)
    co, wo, io = oracle.weighted_kmeans(pts, w, k, r_cpu, warm=warm)
    assert ig == io
    assert np.array_equal(cg, co), np.abs(cg - co).max()
    assert np.array_equal(wg, wo)
    assert r_gpu.next() == r_cpu.next()  # the same number of draws was consumed


def test_weighted_kmeans_reseeds_empty_clusters(ctx):
    pts = clustered(5, 60, 8, centres=3)
    w = np.ones(60, np.float32)
    warm = np.repeat(pts[:1], 4, axis=0)  # duplicated warm centres: clusters 1-3 start empty
    r_gpu, r_cpu = oracle.MT64(9), oracle.MT64(9)
    cg, wg, ig = ctx.weighted_kmeans(pts, w, 4, gen(r_gpu), warm=warm)
    co, wo, io = oracle.weighted_kmeans(pts, w, 4, r_cpu, warm=warm)
    assert ig == io and np.array_equal(cg, co) and np.array_equal(wg, wo)
    assert float(wg.sum()) == 60.0


def test_weighted_kmeans_python_generator(ctx):
    """A Python callable as the generator (the C++ header passes std::mt19937_64 the same way)."""
    pts = clustered(3, 50, 8)
    w = np.ones(50, np.float32)
    r1, r2 = oracle.MT64(77), oracle.MT64(77)
    cg, wg, _ = ctx.weighted_kmeans(pts, w, 5, r1.uniform01)
    co, wo, _ = oracle.weighted_kmeans(pts, w, 5, r2)
    assert np.array_equal(cg, co) and np.array_equal(wg, wo)


def test_weighted_kmeans_rejects_k0(ctx):
    with pytest.raises(_capi.InvalidArgument):
        ctx.weighted_kmeans(np.zeros((3, 2), np.float32), np.ones(3, np.float32), 0, lambda: 0.5)


def make_session(ctx, k, df, ds=8):
    cfg = api.default_config()
    intr = api.make_intrinsics(50, 50, 16, 16, 32, 32)
    s = api.Session(ctx, cfg, 16, ds, k, df, intr)
    g = np.random.default_rng(0)
    atoms = np.zeros((k, df), np.float32)
    s.set_dictionary(atoms, atoms.copy(), g.standard_normal((ds, df)).astype(np.float32))
    return s


def test_session_stream_kmeans_matches_oracle(ctx):
    """Twelve keyframes of dictionary maintenance (pipeline.cpp:201-205): atoms, atom weights and
    the anchor follow the oracle exactly; mass is conserved (integer-valued, exact)."""
    K, df = 32, 64
    s = make_session(ctx, K, df)
    atoms = np.zeros((K, df), np.float32)
    anchor = np.zeros((K, df), np.float32)
    w = np.zeros(K, np.float32)
    r_gpu, r_cpu = oracle.MT64(14), oracle.MT64(14)
    g = np.random.default_rng(14)
    total = 0
    for step in range(12):
        n = 5 + int(g.integers(0, 40))
        batch = clustered(100 + step, n, df, centres=8)
        batch /= np.linalg.norm(batch, axis=1, keepdims=True)  # normalize_embedding_rows
        s.stream_kmeans(batch, gen(r_gpu), decay=0.9 if step % 2 else 1.0)
        oracle.stream_kmeans_update(batch, atoms, anchor, w, r_cpu, decay=0.9 if step % 2 else 1.0)
        total += n
        a_gpu, _ = s.get_dictionary()
        assert np.array_equal(a_gpu, atoms), (step, np.abs(a_gpu - atoms).max())
        assert np.array_equal(s.dict_weights(), w), step
    assert np.array_equal(anchor, atoms)
    s.stream_kmeans(np.zeros((0, df), np.float32), gen(r_gpu))  # empty batch: no-op
    assert np.array_equal(s.get_dictionary()[0], atoms)


def test_session_dict_weights_api(ctx):
    """DictionaryState::weights through the session: the maintained mass, the setter, the >= 0
    check."""
    K, df = 16, 32
    s = make_session(ctx, K, df)
    batch = clustered(1, 20, df)
    s.stream_kmeans(batch, lambda: 0.25)
    w = s.dict_weights()
    assert float(w.sum()) == 20.0 and (w >= 0).all()
    s2 = make_session(ctx, K, df)
    s2.set_dict_weights(w)
    assert np.array_equal(s2.dict_weights(), w)
    with pytest.raises(_capi.InvalidArgument):
        s2.set_dict_weights(-np.ones(K, np.float32))


def test_stream_kmeans_config4_scale(ctx):
    """BASELINE config-4 dictionary (K = 1024, d_f = 1024) with 128-row keyframes: K atoms, exact
    mass, every centre finite; runs in well under a second per keyframe on the device."""
    import time
    K, df = 1024, 1024
    s = make_session(ctx, K, df)
    r = oracle.MT64(4)
    total = 0
    times = []
    for step in range(3):
        batch = clustered(200 + step, 128, df, centres=40)
        batch /= np.linalg.norm(batch, axis=1, keepdims=True)
        t0 = time.perf_counter()
        s.stream_kmeans(batch, gen(r))
        times.append(time.perf_counter() - t0)
        total += 128
        w = s.dict_weights()
        assert float(w.astype(np.float64).sum()) == total
        assert np.isfinite(s.get_dictionary()[0]).all()
    print("stream_kmeans K=1024 d_f=1024 per keyframe (s):", [round(t, 4) for t in times])
