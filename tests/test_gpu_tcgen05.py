"""Pins the hand-written tcgen05 / TMEM conventions (tc_common.cuh) against torch: one-tile
UMMA GEMMs with K-major and MN-major shared-memory operands."""
import ctypes as C

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_12314_b200 import api  # noqa: E402
from paper_2602_12314_b200._capi import check, lib  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return api.Context(0)


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("n,k", [(64, 32), (128, 128), (256, 256), (32, 64)])
def test_umma_tile(ctx, a_mn, b_mn, n, k):
    g = torch.Generator(device="cuda").manual_seed(n * 1000 + k + 10 * a_mn + b_mn)
    a = torch.randn(128, k, device="cuda", generator=g)
    b = torch.randn(n, k, device="cuda", generator=g)
    c = torch.zeros(128, n, device="cuda")
    st = lib().latmap_selftest_umma(ctx.h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()),
                                    C.c_void_p(c.data_ptr()), n, k, a_mn, b_mn)
    check(ctx.h, st)
    torch.cuda.synchronize()
    ref = a.bfloat16().float() @ b.bfloat16().float().T
    err = (c - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, err
