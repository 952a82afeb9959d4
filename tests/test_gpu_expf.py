"""The kernels' std::exp(float) (csrc/expf_ref.h: glibc's expf restated in double arithmetic; used
for every exact-mode / decision-bearing exp: projection scales, sigmoid, the blend's
alpha' = alpha exp(-rho/2), proj/src/render.cpp:54,193,303) equals the libm expf the reference
calls — on ALL 2^32 float bit patterns (NaNs compared as NaNs)."""
import os

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_12314_b200 import api  # noqa: E402
from paper_2602_12314_b200._capi import check, lib  # noqa: E402
import ctypes as C  # noqa: E402


def test_device_expf_equals_libm_on_every_float():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = api.Context(0)
    chunk = 1 << 27
    out = torch.empty(chunk, dtype=torch.float32, device="cuda:0")
    threads = os.cpu_count() or 1
    bad = 0
    for first in range(0, 1 << 32, chunk):
        check(ctx.h, lib().latmap_selftest_expf(ctx.h, first, chunk, C.c_void_p(out.data_ptr())))
        ctx.sync()
        dev = out.cpu().numpy()
        host = oracle.expf_bits(first, chunk, threads)
        diff = dev.view(np.uint32) != host.view(np.uint32)
        diff &= ~(np.isnan(dev) & np.isnan(host))
        bad += int(diff.sum())
        assert bad == 0, (hex(first + int(np.argmax(diff))), dev[np.argmax(diff)], host[np.argmax(diff)])
