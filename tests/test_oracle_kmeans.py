"""Oracle pin for streaming k-means dictionary maintenance: the C
restatement of weighted_kmeans / stream_kmeans_update (proj/src/stream_kmeans.cpp:94-196) against
the properties the reference's own suite checks (proj/tests/test_dictionary.cpp:198-278), and the
generator it consumes (std::mt19937_64 + std::uniform_real_distribution<double>) against the C++
standard's known answer and libstdc++ itself."""
import shutil
import subprocess

import numpy as np
import pytest

import oracle


def test_mt19937_64_known_answer():
    # [rand.predef]: the 10000th invocation of a default-constructed mt19937_64 yields 9981545732273789042
    r = oracle.MT64()
    for _ in range(9999):
        r.next()
    assert r.next() == 9981545732273789042


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ missing")
def test_uniform01_matches_libstdcxx(tmp_path):
    src = tmp_path / "u.cpp"
    src.write_text(r'''
#include <cstdio>
#include <random>
int main() {
  for (unsigned long long seed : {12ULL, 13ULL, 14ULL, 5489ULL}) {
    std::mt19937_64 r(seed);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    for (int i = 0; i < 64; ++i) std::printf("%.17g\n", u(r));
  }
}''')
    exe = tmp_path / "u"
    subprocess.run(["g++", "-O2", str(src), "-o", str(exe)], check=True)
    ref = [float(x) for x in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    mine = []
    for seed in (12, 13, 14, 5489):
        r = oracle.MT64(seed)
        mine += [r.uniform01() for _ in range(64)]
    assert mine == ref


def _state(k, dim, dt):
    return np.zeros((k, dim), dt), np.zeros((k, dim), dt), np.zeros(k, dt)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_virgin_dictionary_absorbs_small_batch(dt):
    # test_dictionary.cpp:198-220: K=8, batch of 5
    rng = oracle.MT64(12)
    batch = np.random.default_rng(12).standard_normal((5, 4)).astype(dt)
    atoms, anchor, w = _state(8, 4, dt)
    oracle.stream_kmeans_update(batch, atoms, anchor, w, rng)
    assert atoms.shape == (8, 4)
    for r in range(5):
        assert np.min(np.linalg.norm(atoms.astype(np.float64) - batch[r], axis=1)) < 1e-9
    assert float(w.sum()) == pytest.approx(5.0)
    assert int((w == 0).sum()) == 3  # the filled-to-K duplicates carry zero weight
    assert np.array_equal(anchor, atoms)


def test_two_separated_clusters_recover_means():
    # test_dictionary.cpp:222-250
    rng = oracle.MT64(13)
    g = np.random.default_rng(13)
    mu = [np.zeros(4), np.full(4, 10.0)]
    batch = np.stack([mu[r % 2] + g.normal(0, 0.01, 4) for r in range(60)])
    atoms, anchor, w = _state(2, 4, np.float64)
    oracle.stream_kmeans_update(batch, atoms, anchor, w, rng)
    ma = batch[batch.sum(1) < 20].mean(0)
    mb = batch[batch.sum(1) >= 20].mean(0)
    near0, near1 = (ma, mb) if np.linalg.norm(atoms[0] - ma) < np.linalg.norm(atoms[0] - mb) else (mb, ma)
    assert np.linalg.norm(atoms[0] - near0) < 0.05
    assert np.linalg.norm(atoms[1] - near1) < 0.05
    assert float(w.sum()) == pytest.approx(60.0)
    before = atoms.copy()
    oracle.stream_kmeans_update(batch, atoms, anchor, w, rng)  # identical batch: atoms stay, weights double
    assert np.abs(atoms - before).max() < 1e-6
    assert float(w.sum()) == pytest.approx(120.0)


def test_size_stays_k_and_mass_is_conserved():
    # test_dictionary.cpp:253-269 (float, integer-valued mass is exact)
    rng = oracle.MT64(14)
    g = np.random.default_rng(14)
    atoms, anchor, w = _state(16, 6, np.float32)
    total = 0
    for _ in range(12):
        n = 5 + int(g.integers(0, 40))
        batch = g.standard_normal((n, 6)).astype(np.float32)
        oracle.stream_kmeans_update(batch, atoms, anchor, w, rng)
        total += n
        assert atoms.shape == (16, 6)
        assert float(w.astype(np.float64).sum()) == total
        assert w.min() >= 0


def test_empty_batch_is_noop():
    # test_dictionary.cpp:271-278
    rng = oracle.MT64(15)
    g = np.random.default_rng(15)
    atoms = g.standard_normal((4, 5))
    anchor = atoms.copy()
    w = np.ones(4)
    a0, w0 = atoms.copy(), w.copy()
    oracle.stream_kmeans_update(np.zeros((0, 5)), atoms, anchor, w, rng)
    assert np.array_equal(atoms, a0) and np.array_equal(w, w0)


def test_weighted_kmeans_warm_start_reseed_and_ties():
    """Warm-started centres fill the first rows; a duplicated warm centre leaves a cluster empty
    (re-seeded at the heaviest unclaimed point); ties in the assignment go to the lower index."""
    rng = oracle.MT64(3)
    pts = np.array([[0, 0], [0, 0.1], [5, 5], [5, 5.1], [9, 0]], np.float64)
    w = np.array([1, 2, 1, 3, 0.5])
    warm = np.array([[0, 0], [0, 0]], np.float64)  # duplicate: centre 1 gets no points
    cen, cw, it = oracle.weighted_kmeans(pts, w, 3, rng, warm=warm)
    assert it >= 2
    assert float(cw.sum()) == pytest.approx(float(w.sum()))
    # every point is within its centre's cluster: masses cover {0,1}, {2,3} and {4} in some order
    assert sorted(np.round(cw, 6).tolist()) == sorted([3.0, 4.0, 0.5])
    # exact tie: two identical centres, the lower index wins every point
    c2, w2, _ = oracle.weighted_kmeans(np.array([[1.0, 1.0]]), np.array([1.0]), 2, oracle.MT64(4),
                                       warm=np.array([[1.0, 1.0], [1.0, 1.0]]), max_iters=1)
    assert w2.tolist() == [1.0, 0.0]
