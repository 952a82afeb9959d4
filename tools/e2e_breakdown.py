import os, sys
"""Host-side breakdown of one e2e step on config 2 (set_frames / step launch / loss read)."""
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time

import numpy as np
import torch

from paper_2602_12314_b200 import api, synthetic
import bench

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
s.set_batch(len(pinned))
for _ in range(5):
    s.step(read=True)
torch.cuda.synchronize()
T = {"set_frames": [], "step_launch": [], "read": [], "total": []}
for _ in range(20):
    t0 = time.perf_counter()
    s.set_frames(pinned)
    t1 = time.perf_counter()
    s.step(read=False)
    t2 = time.perf_counter()
    s.read_loss()
    t3 = time.perf_counter()
    T["set_frames"].append(t1 - t0), T["step_launch"].append(t2 - t1), T["read"].append(t3 - t2), T["total"].append(t3 - t0)
print({k: round(1e3 * float(np.median(v)), 3) for k, v in T.items()})

# split set_frames: Python argument marshalling vs the C call
import ctypes as C
from paper_2602_12314_b200._capi import Frame, lib, check
cf = (Frame * len(pinned))()
for i, f in enumerate(pinned):
    cf[i] = Frame(api.make_pose(f.pose_rot, f.pose_trans), s._np_ptr(f.rgb), s._np_ptr(f.depth),
                  s._np_ptr(f.assignment), s._np_ptr(f.features), f.features.shape[0])
tc = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    check(ctx.h, lib().latmap_session_set_frames(s.h, len(pinned), cf))
    tc.append(time.perf_counter() - t0)
print({"c_set_frames_ms": round(1e3 * float(np.median(tc)), 3)})
