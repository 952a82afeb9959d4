"""Stream scheduling of the Stage-I step against the plain schedule, bit for bit.

Early colour / feature Adam (latmap_session_step): once the last frame's render backward is
done, the colour and feature blocks -- whose gradients K8 writes directly -- are updated on the
render stream while the projection backward, the decoder's step-end reduce and the trust term
run on the context stream; the remaining blocks follow (csrc/capi.cu session_objective /
session_adam). Against LATMAP_EARLY_CF=0 (all eight blocks after the objective) the step is the
same arithmetic, so in deterministic mode the parameters, the gradient buffer and the losses are
bit-identical after several steps, through the captured graph and through direct launches. The
comparison run also puts every render on one render stream (LATMAP_RSTREAMS=1) and the image
losses back on the context stream (LATMAP_LSTREAM=0), so the two-render-stream and loss-stream
schedules are covered by the same equality. Each variant runs in its own process (the switches
are read once)."""
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
s.set_graphs(sys.argv[2] == "1")
losses = []
for _ in range(4):
    l = s.step()
    losses += [l[k] for k in ("l_rgb", "l_depth", "l_cos", "total")]
np.save(sys.argv[1], np.concatenate([s.params_buffer().cpu().numpy(), s.grad_buffer().cpu().numpy(),
                                     np.array(losses, np.float32)]))
"""


@pytest.mark.parametrize("graphs", ["1", "0"])
def test_early_colour_feature_adam_bit_identical(tmp_path, graphs):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    outs = []
    for mode in ("1", "0"):
        f = tmp_path / f"p{mode}.npy"
        env = dict(os.environ, LATMAP_EARLY_CF=mode, LATMAP_LSTREAM=mode, LATMAP_RSTREAMS="2" if mode == "1" else "1")
        subprocess.run([sys.executable, "-c", SCRIPT % ROOT, str(f), graphs], env=env, check=True, timeout=600)
        outs.append(np.load(f))
    assert np.array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
