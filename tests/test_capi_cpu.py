"""CPU-side checks of the boundary: the C-ABI library loads, exports every entry point
include/latmap_b200.h declares, and refuses to run without a GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2602_12314_b200 import _capi, synthetic

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "latmap_b200.h")).read()
    return sorted(set(re.findall(r"\b(latmap_[a-z_0-9]+)\s*\(", txt)))


def test_header_and_binding_agree():
    syms = header_symbols()
    assert len(syms) >= 30
    assert sorted(_capi.EXPORTED) == syms


def test_library_exports_every_symbol():
    L = _capi.lib()
    missing = [s for s in header_symbols() if not hasattr(L, s)]
    assert not missing, missing


def test_struct_layouts_match_header():
    assert C.sizeof(_capi.ProjectedSplat) == 52
    assert C.sizeof(_capi.Intrinsics) == 24
    assert C.sizeof(_capi.Pose) == 28
    assert C.sizeof(_capi.LossBreakdown) == 7 * 4 + 4 + 8 + 8  # padding before int64
    cfg = _capi.Config()
    _capi.lib().latmap_default_config(C.byref(cfg))
    assert cfg.lambda_feat == pytest.approx(5.0) and cfg.lambda_i2 == pytest.approx(0.8) and cfg.dict_learn == 1


def test_no_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = _capi.lib().latmap_ctx_create(0, None, C.byref(h))
    assert st == _capi.ECUDA
    with pytest.raises(_capi.LatmapError):
        _capi.check(None, st)


def test_synthetic_generator_is_seeded_and_shaped():
    calls = []

    def fake_render(m, q, t, intr):
        calls.append((q, t))
        return (np.zeros((intr.height, intr.width, 3)), np.ones((intr.height, intr.width)),
                np.ones((intr.height, intr.width)))

    a = synthetic.make_workload(2, fake_render, scale=0.125)
    b = synthetic.make_workload(2, fake_render, scale=0.125)
    assert len(a.frames) == 8 and len(calls) == 16
    assert np.array_equal(a.map.positions, b.map.positions)
    f = a.frames[0]
    assert f.assignment.shape == (a.intr.height, a.intr.width) and f.assignment.max() < f.features.shape[0]
    np.testing.assert_allclose(np.linalg.norm(f.features, axis=1), 1.0, rtol=1e-5)
    np.testing.assert_allclose(np.linalg.norm(a.atoms, axis=1), 1.0, rtol=1e-5)
    # camera walk: 0.1 m steps
    steps = [np.linalg.norm(np.subtract(a.frames[i + 1].pose_trans, a.frames[i].pose_trans)) for i in range(7)]
    np.testing.assert_allclose(steps, 0.1, rtol=1e-6)
