"""Shared fixtures restating the reference's test helpers (proj/tests/oracles.hpp)."""
import numpy as np

import oracle


def random_map(n, query_dim, rng, dtype=np.float64, depth_min=1.2, depth_max=3.5):
    """oracle::random_map, oracles.hpp:197-217."""
    pos = np.stack([(rng.random(n) * 2 - 1) * 0.8, (rng.random(n) * 2 - 1) * 0.6,
                    depth_min + rng.random(n) * (depth_max - depth_min)], 1)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    col = rng.random((n, 3))
    lsc = np.log(0.05 + rng.random((n, 3)) * 0.25)
    opa = rng.random(n) * 3 - 1
    feat = rng.standard_normal((n, query_dim)) * 0.5
    return oracle.GaussianMap(*[np.ascontiguousarray(a, dtype) for a in (pos, q, col, lsc, opa, feat)])


def small_intrinsics(w=16, h=16, f=20.0):
    """oracle::small_intrinsics, oracles.hpp:219-227."""
    return oracle.make_intr(f, f, w / 2, h / 2, w, h)


def grad_check(loss, block, analytic, step=1e-4, max_coords=0):
    """grad_check, obj/grad_check.hpp:23-47 (central differences, |ga-gfd|/(|gfd|+1e-8))."""
    flat = block.reshape(-1)
    an = np.asarray(analytic).reshape(-1)
    count = flat.size
    stride = 1
    if max_coords > 0 and count > max_coords:
        stride = (count + max_coords - 1) // max_coords
    worst = 0.0
    for i in range(0, count, stride):
        saved = flat[i]
        flat[i] = saved + step
        up = loss()
        flat[i] = saved - step
        down = loss()
        flat[i] = saved
        fd = (up - down) / (2 * step)
        rel = abs(an[i] - fd) / (abs(fd) + 1e-8)
        worst = max(worst, rel)
    return worst
