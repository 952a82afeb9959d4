import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2602_12314_b200 import api, synthetic
ctx = api.Context(0)
st = synthetic.make_streaming(n_global=1_000_000, nframes=1, scale=0.1, device="cuda")
intr = api.make_intrinsics(st.intr.fx, st.intr.fy, st.intr.cx, st.intr.cy, st.intr.width, st.intr.height)
print("image", st.intr.width, st.intr.height)
store = api.Store(ctx, st.capacity, 32)
store.insert_global(st.records, st.voxel_size)
q, t = st.poses[0]
org, rows = store.fetch_local(np.asarray(t, np.float32), st.radius, gather=True)
print("rows", rows.shape)
gm = api.GaussianMap(rows[:, 0:3].contiguous(), rows[:, 3:7].contiguous(), rows[:, 7:10].contiguous(), rows[:, 10:13].contiguous(), rows[:, 13].contiguous(), rows[:, 14:].contiguous())
out = api.render(ctx, gm, api.make_pose(q, t), intr)
frame = synthetic.Frame(q, t, out.color.cpu().numpy() * 0.9, out.depth.cpu().numpy(), st.assignments[0], st.features[0])
cfg = api.default_config(**st.lambdas)
s = api.Session(ctx, cfg, 0, 32, 256, 1024, intr)
s.set_dictionary(st.atoms, st.atoms, st.proj)
s.import_rows(rows.contiguous())
s.set_frames([frame]); s.set_batch(1)
s.step(read=True)
print("nondet ok", s.stats(1))
ctx.set_deterministic(True)
try:
    s.step(read=True)
    print("det ok")
except Exception as e:
    print("det fail", e)
    import ctypes
    print(torch.cuda.memory_allocated(), torch.cuda.mem_get_info())
