"""The REFERENCE ITSELF, compiled here (oracle/ref/Makefile: /root/reference/proj/src unmodified,
against the from-scratch Eigen / doctest stand-ins in oracle/stand_ins), pins the oracle
restatement that the GPU parity tests use:

  * the reference's own seven doctest suites run green on the stand-ins (the six hot-path suites
    entirely; test_io has four cases that fail in the reference itself, listed below with why);
  * the C restatement (oracle/latmap_oracle.c) equals the compiled reference BIT FOR BIT on the
    BASELINE config-0 and config-2 workloads: rendered images, every LossBreakdown term, every
    gradient block, and the map / dictionary after Adam steps.

Skipped where oracle/_ref was not built (the GPU box builds nothing; the driver's CPU run here
builds it from /root/reference in __graft_entry__.build()).
"""
import os
import subprocess

import numpy as np
import pytest

import oracle
from oracle import ref
from paper_2602_12314_b200 import synthetic

REF_DIR = os.path.join(os.path.dirname(oracle.__file__), "_ref")
pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built (needs /root/reference)")

# test_io cases that fail in the reference itself, independent of the Eigen / doctest stand-ins:
KNOWN_REFERENCE_FAILURES = {
    # test_io.cpp:55-57 expects one byte more than write_tensor emits for its own layout
    # (tensor_file.cpp: 4-byte name length + name + dtype + rank + dims + payload per entry)
    "tensor container: typed entries round-trip exactly",
    # test_io.cpp:131: 1 - dot/(|f||f|) for the float row (0.3, 0.3) is -1.8e-8 in float arithmetic
    # (sqrtf(0.18f)^2 != 0.18f), above the 1e-9 bound
    "metric_cos examples",
    # test_io.cpp:292: class 2's box (synthetic.cpp "rooms", seed 42) is behind or outside the
    # view of all six trajectory poses, so no label 2 is ever rendered (pure scalar ray casting)
    "gen_synthetic: deterministic, validates, classes all visible",
    # test_io.cpp:340-346: the ground-truth model (synthetic.cpp:329-364) places floor splats 2 cm in
    # front of the first camera; their 3-sigma footprints cover the whole image (render.cpp:75-91),
    # while the ray caster ignores hits nearer than kRayNear = 5 cm (synthetic.cpp:15,118)
    "evaluate_map on the ground-truth model bypasses learning cleanly",
}


def run_suite(name):
    p = subprocess.run([os.path.join(REF_DIR, name)], cwd=REF_DIR, capture_output=True, text=True, timeout=600)
    failed = {line.split('"')[1] for line in p.stderr.splitlines() if line.strip().startswith("in TEST CASE")}
    return p.returncode, p.stdout + p.stderr, failed


@pytest.mark.parametrize("suite", ["test_core", "test_render", "test_dictionary", "test_losses", "test_objective",
                                   "test_store"])
def test_reference_suite_green(suite):
    rc, out, failed = run_suite(suite)
    assert rc == 0 and not failed, out[-2000:]


def test_reference_io_suite_only_known_failures():
    rc, out, failed = run_suite("test_io")
    assert failed == KNOWN_REFERENCE_FAILURES, out[-3000:]


def _workload(cfg_id, scale):
    def orender(m, q, t, intr):
        om = oracle.GaussianMap(m.positions, m.rotations, m.colors, m.log_scales, m.opacity_logits, m.features)
        o = oracle.render(om, q, t, oracle.make_intr(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height),
                          threads=4)
        return o["color"], o["depth"], o["alpha"]
    return synthetic.make_workload(cfg_id, orender, scale=scale)


def _oracle_side(w):
    om = oracle.GaussianMap(*[np.ascontiguousarray(getattr(w.map, f), np.float32) for f in oracle.FIELDS])
    oi = oracle.make_intr(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height)
    d = oracle.Dictionary(w.atoms.copy(), w.anchor.copy(), w.proj.copy(), np.float32(w.temperature))
    frames = [oracle.Frame(f.pose_rot, f.pose_trans, f.rgb, f.depth, f.assignment.reshape(-1), f.features)
              for f in w.frames]
    cfg = oracle.Config(lambda_l2=w.lambdas["lambda_l2"], lambda_i2=w.lambdas["lambda_i2"],
                        lambda_trust=w.lambdas["lambda_trust"])
    return om, oi, d, frames, cfg


def _ref_cfg(w):
    return ref.make_config(lambda_l2=w.lambdas["lambda_l2"], lambda_i2=w.lambdas["lambda_i2"],
                           lambda_trust=w.lambdas["lambda_trust"])


def _same_bits(a, b):
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.parametrize("cfg_id,scale", [(0, 0.25), (0, 1.0), (2, 0.125)])
def test_oracle_equals_reference_bit_for_bit(cfg_id, scale):
    oracle.set_gemm_threads(os.cpu_count() or 1)
    w = _workload(cfg_id, scale)
    om, oi, d, frames, cfg = _oracle_side(w)
    for f in w.frames[:2]:
        a = oracle.render(om, f.pose_rot, f.pose_trans, oi, threads=4)
        b = ref.render(w.map, f.pose_rot, f.pose_trans, w.intr, threads=4)
        for k in ("color", "depth", "query", "alpha"):
            assert _same_bits(a[k], b[k]), k
    lo, (g, dp, da) = oracle.total_objective(om, d, frames, oi, cfg, threads=4)
    lr, (gr, dpr, dar) = ref.total_objective(w.map, w.atoms, w.anchor, w.proj, w.temperature, w.frames, w.intr,
                                             _ref_cfg(w), threads=4)
    for k in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust", "total", "supervised_rows"):
        assert np.float32(lo[k]).tobytes() == np.float32(lr[k]).tobytes() if k != "supervised_rows" else \
            lo[k] == lr[k], (k, lo[k], lr[k])
    go = np.concatenate([getattr(g, f).reshape(-1) for f in oracle.FIELDS])
    assert _same_bits(go, gr)
    assert _same_bits(dp, dpr) and _same_bits(da, dar)


def test_oracle_adam_steps_equal_reference():
    """Three Stage-I iterations (total_objective + MapOptimizer::step_map + step_dict,
    pipeline.cpp:75-95,236-246) on both sides: identical losses and final state, bit for bit."""
    w = _workload(0, 0.25)
    om, oi, d, frames, cfg = _oracle_side(w)
    rs = ref.Session(w.map, w.atoms, w.anchor, w.proj, w.temperature, w.frames, w.intr, _ref_cfg(w), threads=4)
    opt = oracle.MapOptimizer()
    for _ in range(3):
        lo, (g, dp, da) = oracle.total_objective(om, d, frames, oi, cfg, threads=4)
        opt.step_map(om, g, cfg)
        opt.step_dict(d, dp, da, cfg)
        lr = rs.step()
        assert np.float32(lo["total"]).tobytes() == np.float32(lr["total"]).tobytes(), (lo["total"], lr["total"])
    m_ref, a_ref, p_ref = rs.get()
    m_or = np.concatenate([getattr(om, f).reshape(-1) for f in oracle.FIELDS])
    assert _same_bits(m_or, m_ref)
    assert _same_bits(d.atoms, a_ref) and _same_bits(d.proj, p_ref)
