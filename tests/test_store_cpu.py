"""Host-side voxel key / hash functions of the product library vs the oracle and the
reference's KATs (proj/tests/test_store.cpp:42-64) — no GPU needed."""
import numpy as np

import oracle
from paper_2602_12314_b200 import api


def test_voxel_of_kats():  # test_store.cpp:42-54
    assert api.voxel_of((0.015, -0.003, 0.021), 0.01) == (1, -1, 2)
    assert api.voxel_of((0, 0, 0), 0.01) == (0, 0, 0)
    assert api.voxel_of((0.01, 0.01, 0.01), 0.01) == (1, 1, 1)


def test_hash_kats():  # test_store.cpp:56-64
    assert api.hash_voxel((0, 0, 0), 1 << 20) == 0
    assert api.hash_voxel((1, 0, 0), 1 << 20) == 455773
    for i in range(-5, 0):
        assert api.hash_voxel((i, 2 * i, -7 * i), 4096) >= 0


def test_keys_and_hash_bit_exact_vs_oracle():
    rng = np.random.default_rng(5)
    pts = np.concatenate([rng.uniform(-30, 30, (4000, 3)), rng.uniform(-1e-3, 1e-3, (500, 3)),
                          np.round(rng.uniform(-5, 5, (500, 3)), 2)]).astype(np.float32)
    for vs in (0.01, 0.5, 0.05, 1.0 / 3.0):
        for p in pts[::7]:
            k = api.voxel_of(p, vs)
            assert k == oracle.voxel_of(p, vs)
            for cap in (1 << 24, 4096, 1000003, 64):
                assert api.hash_voxel(k, cap) == oracle.hash_voxel(k, cap)
