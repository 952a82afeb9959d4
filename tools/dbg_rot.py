import sys, os, numpy as np
sys.path.insert(0, "/root/repo")
import torch, oracle
from paper_2602_12314_b200 import api, synthetic
from tests.test_gpu_decoder_oracle import oracle_render_fn, run_oracle, THREADS
oracle.set_gemm_threads(THREADS)
ctx = api.Context(0)
w = synthetic.make_workload(2, oracle_render_fn, scale=0.25)
for prec in (0, 1):
    cfg = api.default_config(**w.lambdas); cfg.decoder_precision = prec
    intr = api.make_intrinsics(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height)
    s = api.Session(ctx, cfg, w.map.n, w.map.features.shape[1], w.atoms.shape[0], w.atoms.shape[1], intr)
    s.set_map(w.map); s.set_dictionary(w.atoms, w.anchor, w.proj); s.set_frames(w.frames); s.set_batch(len(w.frames))
    loss = s.objective(want_grad=True); gb = s.grad_buffer().cpu().numpy().copy()
    ref, (g, dp, da) = run_oracle(w)
    n = w.map.n
    for nm, off, cnt in (("positions",0,3*n),("rotations",3*n,4*n),("colors",7*n,3*n),("log_scales",10*n,3*n),("opacity",13*n,n)):
        a = gb[off:off+cnt]; b = getattr(g, oracle.FIELDS[["positions","rotations","colors","log_scales","opacity"].index(nm)]).reshape(-1)
        print(prec, nm, np.linalg.norm(a-b)/np.linalg.norm(b), np.linalg.norm(a), np.linalg.norm(b))
    # single frames
    for b in range(len(w.frames)):
        s1 = api.Session(ctx, cfg, w.map.n, w.map.features.shape[1], w.atoms.shape[0], w.atoms.shape[1], intr)
        s1.set_map(w.map); s1.set_dictionary(w.atoms, w.anchor, w.proj); s1.set_frames([w.frames[b]]); s1.set_batch(1)
        s1.objective(want_grad=True); g1 = s1.grad_buffer().cpu().numpy().copy()
        w1 = synthetic.Workload(**{**w.__dict__, "frames": [w.frames[b]]}) if False else None
        om = oracle.GaussianMap(*[np.ascontiguousarray(getattr(w.map, f), np.float32) for f in oracle.FIELDS])
        d = oracle.Dictionary(w.atoms.copy(), w.anchor.copy(), w.proj.copy(), np.float32(w.temperature))
        f = w.frames[b]
        fr = [oracle.Frame(f.pose_rot, f.pose_trans, f.rgb, f.depth, f.assignment.reshape(-1), f.features)]
        c = oracle.Config(lambda_l2=0.0, lambda_i2=0.0, lambda_trust=w.lambdas["lambda_trust"])
        _, (gg, _, _) = oracle.total_objective(om, d, fr, oracle.make_intr(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height), c, threads=THREADS)
        a = g1[3*n:7*n]; bb = gg.rotations.reshape(-1)
        print("  frame", b, f.pose_rot, "rot err", np.linalg.norm(a-bb)/np.linalg.norm(bb), "pos err", np.linalg.norm(g1[:3*n]-gg.positions.reshape(-1))/np.linalg.norm(gg.positions))
    break
