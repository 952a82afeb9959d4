"""Host/device breakdown of one config-3 streaming frame (export, store sync, import, set_frames,
10 Stage-I steps), each phase bracketed by a device synchronize."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_12314_b200 import api, synthetic

torch.cuda.set_device(0)
ctx = api.Context(0)
nfr = 6
st = synthetic.make_streaming(nframes=nfr, device="cuda")
intr = api.make_intrinsics(st.intr.fx, st.intr.fy, st.intr.cx, st.intr.cy, st.intr.width, st.intr.height)
store = api.Store(ctx, st.capacity, 32)
store.insert_global(st.records, st.voxel_size)
del st.records
frames = []
for f, (q, t) in enumerate(st.poses):
    frames.append(synthetic.Frame(q, t, np.zeros((st.intr.height, st.intr.width, 3), np.float32),
                                  np.zeros((st.intr.height, st.intr.width), np.float32), st.assignments[f],
                                  st.features[f]))
cfg = api.default_config(**st.lambdas)
cfg.decoder_precision = 1
s = api.Session(ctx, cfg, 0, 32, st.atoms.shape[0], st.atoms.shape[1], intr)
s.set_dictionary(st.atoms, st.atoms, st.proj)
origin = np.zeros(0, np.int64)
for f in range(nfr):
    T = {}
    q, t = st.poses[f]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rows = s.export_rows() if s.n else None
    torch.cuda.synchronize(); T["export"] = time.perf_counter() - t0; t0 = time.perf_counter()
    d_out, origin_new, kept, stats = store.sync(rows, origin, np.ones(len(origin), np.uint8),
                                                np.asarray(t, np.float32), st.radius, st.voxel_size)
    torch.cuda.synchronize(); T["store_sync"] = time.perf_counter() - t0; t0 = time.perf_counter()
    s.import_rows(d_out.contiguous(), kept=kept if len(origin) else None)
    origin = origin_new
    torch.cuda.synchronize(); T["import"] = time.perf_counter() - t0; t0 = time.perf_counter()
    s.set_frames([frames[f]])
    s.set_batch(1)
    torch.cuda.synchronize(); T["set_frames"] = time.perf_counter() - t0; t0 = time.perf_counter()
    s.step(read=False)
    torch.cuda.synchronize(); T["step1"] = time.perf_counter() - t0; t0 = time.perf_counter()
    for _ in range(st.iters_per_frame - 1):
        s.step(read=False)
    torch.cuda.synchronize(); T["steps2_10"] = time.perf_counter() - t0
    print(f, {k: round(1e3 * v, 2) for k, v in T.items()}, "active", s.n, flush=True)
