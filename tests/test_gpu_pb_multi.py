"""The projection backward of all keyframes in one pass (render_project_backward_multi, the
session default) against one K9 launch per frame (LATMAP_PB_MULTI=0): the same float additions
in the same frame order, so in deterministic mode the rendered images, the loss terms and the
gradient buffers are bit-identical. Each variant runs in its own process (the switch is read
once)."""
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_2602_12314_b200 import api, synthetic
ctx = api.Context(0)
def rend(m, q, t, intr):
    out = api.render(ctx, api.GaussianMap.from_numpy(m), api.make_pose(q, t),
                     api.make_intrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
    return out.color.cpu().numpy(), out.depth.cpu().numpy(), out.alpha.cpu().numpy()
w = synthetic.make_workload(2, rend, scale=0.25)
cfg = api.default_config(**w.lambdas)
cfg.decoder_precision = 1
intr = api.make_intrinsics(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height)
s = api.Session(ctx, cfg, w.map.n, w.map.features.shape[1], w.atoms.shape[0], w.atoms.shape[1], intr)
s.set_map(w.map); s.set_dictionary(w.atoms, w.anchor, w.proj); s.set_frames(w.frames); s.set_batch(len(w.frames))
ctx.set_deterministic(True)
s.objective(want_grad=True)
s.objective(want_grad=True)
loss = s.objective(want_grad=True)
imgs = [t.cpu().numpy().ravel() for b in range(len(w.frames)) for t in s.frame_images(b) if t is not None]
np.save(sys.argv[1], np.concatenate([s.grad_buffer().cpu().numpy()] + imgs
                                    + [np.array([loss[k] for k in ("l_rgb", "l_depth", "l_cos", "total")], np.float32)]))
"""


def test_multi_frame_projection_backward_bit_identical(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    outs = []
    for mode in ("1", "0"):
        f = tmp_path / f"g{mode}.npy"
        env = dict(os.environ, LATMAP_PB_MULTI=mode)
        subprocess.run([sys.executable, "-c", SCRIPT % ROOT, str(f)], env=env, check=True, timeout=600)
        outs.append(np.load(f))
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
