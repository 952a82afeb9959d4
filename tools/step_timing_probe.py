"""Probe: config-2 step time under different host submission patterns (development tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_12314_b200 import api, synthetic  # noqa: E402

ctx = api.Context(0)
w = synthetic.make_workload(2, bench.gpu_render_fn(ctx))
cfg = api.default_config(**w.lambdas)
cfg.decoder_precision = 1
intr = api.make_intrinsics(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height)
s = api.Session(ctx, cfg, w.map.n, w.map.features.shape[1], w.atoms.shape[0], w.atoms.shape[1], intr)
s.set_map(w.map)
s.set_dictionary(w.atoms, w.anchor, w.proj)
pinned = [synthetic.Frame(f.pose_rot, f.pose_trans, *[torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
                                                       for a in (f.rgb, f.depth, f.assignment, f.features)])
          for f in w.frames]
s.set_frames(pinned)
s.set_batch(8)
stream = torch.cuda.current_stream()
for _ in range(5):
    s.step(read=False)
torch.cuda.synchronize()


def timed(name, body, n=30):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for k in range(n):
        body(k)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1000
    print(f"{name:40s} {1000 * n / e0.elapsed_time(e1):8.2f} it/s (events)  {1000 * n / wall:8.2f} it/s (wall)",
          flush=True)


ev = [torch.cuda.Event() for _ in range(2)]
timed("back to back", lambda k: s.step(read=False))
timed("back to back (again)", lambda k: s.step(read=False))


def lagged(k):
    s.step(read=False)
    ev[k % 2].record(stream)
    if k:
        ev[(k - 1) % 2].synchronize()


timed("one step in flight (sync k-1)", lagged)


def setf(k):
    s.set_frames(pinned)
    s.step(read=False)


timed("set_frames + step, back to back", setf)


def setf_lag(k):
    s.set_frames(pinned)
    lagged(k)


timed("set_frames + step, sync k-1", setf_lag)
timed("back to back (after)", lambda k: s.step(read=False))
