"""Standalone reconstruct on the tensor cores (latmap_ctx_set_reconstruct_precision(ctx, 1)):
DL1's bf16 attention tiles times D on tcgen05 (decoder_dl.cu dl_rec_kernel), the path
evaluate_map / query_map take (proj/src/evaluate.cpp:41,80; reconstruct,
proj/src/dictionary.cpp:25-53). Checked against the oracle per row: the north-star bar is a
decoded-embedding cosine >= 0.999; bf16 operands with fp32 accumulation (the logits S = Q Kd^T
in bf16, as the configs' decoder computes them) give a median row cosine of about 0.99999 and a
worst row above 0.9998 on these problems; the asserted bars are cos >= 0.9995 and a row relative
error <= 3e-2. Unsupported shapes (K = 128) fall back to the fp32 path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2602_12314_b200 import api  # noqa: E402

ROW_COS = 0.9995
ROW_REL = 3e-2


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = api.Context(0)
    yield c
    c.set_reconstruct_precision(0)


def problem(seed, n, ds, k, df):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((n, ds)).astype(np.float32)
    atoms = (rng.standard_normal((k, df)) / np.sqrt(df)).astype(np.float32)
    proj = (rng.standard_normal((ds, df)) * (2.0 / np.sqrt(ds))).astype(np.float32)
    return q, atoms, proj


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


@pytest.mark.parametrize("n,ds,k,df", [(5000, 32, 256, 512), (4133, 64, 1024, 1024), (777, 32, 512, 768),
                                       (129, 64, 256, 256)])
def test_reconstruct_tc_matches_oracle(ctx, n, ds, k, df):
    q, atoms, proj = problem(n + k, n, ds, k, df)
    temp = 0.7
    ref = oracle.reconstruct(q, atoms, proj, temp).astype(np.float64)
    ctx.set_reconstruct_precision(1)
    try:
        got = api.reconstruct(ctx, dev(q), dev(atoms), dev(proj), temp).cpu().numpy().astype(np.float64)
    finally:
        ctx.set_reconstruct_precision(0)
    assert np.isfinite(got).all()
    cos = (got * ref).sum(1) / (np.linalg.norm(got, axis=1) * np.linalg.norm(ref, axis=1))
    rel = np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)
    assert cos.min() >= ROW_COS, cos.min()
    assert rel.max() <= ROW_REL, rel.max()
    # and it is not the fp32 path: the bf16 rounding shows
    fp32 = api.reconstruct(ctx, dev(q), dev(atoms), dev(proj), temp).cpu().numpy().astype(np.float64)
    assert np.abs(fp32 - ref).max() < np.abs(got - ref).max()


def test_reconstruct_tc_unsupported_shape_falls_back(ctx):
    q, atoms, proj = problem(3, 300, 32, 128, 768)  # K = 128 (config 1): fp32 path
    a = api.reconstruct(ctx, dev(q), dev(atoms), dev(proj), 1.0).cpu().numpy()
    ctx.set_reconstruct_precision(1)
    try:
        b = api.reconstruct(ctx, dev(q), dev(atoms), dev(proj), 1.0).cpu().numpy()
    finally:
        ctx.set_reconstruct_precision(0)
    # the fp32 path both times (its split-K sums may differ in the last bit run to run)
    np.testing.assert_allclose(b, a, rtol=1e-5, atol=1e-7)


def test_query_map_tc(ctx):
    """query_map (evaluate.hpp:37-40) over 20000 Gaussians with the tcgen05 reconstruct."""
    n, ds, k, df = 20000, 32, 256, 512
    q, atoms, proj = problem(11, n, ds, k, df)
    emb = np.random.default_rng(12).standard_normal(df).astype(np.float32)
    rec = oracle.reconstruct(q, atoms, proj, 1.0).astype(np.float64)
    ref = rec @ emb / (np.linalg.norm(rec, axis=1) * np.linalg.norm(emb))
    ctx.set_reconstruct_precision(1)
    try:
        got = api.query_map(ctx, dev(q), dev(atoms), dev(proj), 1.0, dev(emb)).cpu().numpy()
    finally:
        ctx.set_reconstruct_precision(0)
    np.testing.assert_allclose(got, ref, atol=5e-3)
