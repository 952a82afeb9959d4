#!/usr/bin/env python
"""One small Stage-I step per kernel family, for compute-sanitizer (memcheck / racecheck /
synccheck) on the GPU box:

  compute-sanitizer --tool memcheck   python tools/sanitize_run.py
  compute-sanitizer --tool racecheck  python tools/sanitize_run.py

config 0 (fp32 SIMT decoder, K1-K5/K8-K10), config 2 at 1/8 scale (fused tcgen05 DEC1/DEC2),
config 2 forced onto the staged path and config 4 at 1/8 scale (DL1-DL5, TMA tensor maps).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2602_12314_b200 import api, synthetic  # noqa: E402


def gpu_render(ctx):
    def fn(m, q, t, intr):
        out = api.render(ctx, api.GaussianMap.from_numpy(m), api.make_pose(q, t),
                         api.make_intrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
        return out.color.cpu().numpy(), out.depth.cpu().numpy(), out.alpha.cpu().numpy()
    return fn


def main():
    ctx = api.Context(0)
    for cfg_id, scale, path in ((0, 0.25, 0), (2, 0.125, 0), (2, 0.125, 2), (4, 0.125, 0)):
        w = synthetic.make_workload(cfg_id, gpu_render(ctx), scale=scale)
        ctx.set_decoder_path(path)
        cfg = api.default_config(**w.lambdas)
        cfg.decoder_precision = 0 if cfg_id == 0 else 1
        intr = api.make_intrinsics(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height)
        s = api.Session(ctx, cfg, w.map.n, w.map.features.shape[1], w.atoms.shape[0], w.atoms.shape[1], intr)
        s.set_map(w.map)
        s.set_dictionary(w.atoms, w.anchor, w.proj)
        s.set_frames(w.frames)
        s.set_batch(len(w.frames))
        s.set_graphs(False)  # plain launches (the sanitizer attributes reports per kernel launch)
        loss = s.step(read=True)
        print(f"config {cfg_id} scale {scale} path {path}: total {loss['total']:.6f}", flush=True)
        del s
    ctx.set_decoder_path(0)
    ctx.sync()
    print("sanitize_run: done", flush=True)


if __name__ == "__main__":
    main()
