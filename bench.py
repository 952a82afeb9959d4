#!/usr/bin/env python
"""Benchmark: latent-map optimisation iterations/s (render + dict-attention decode + backward
+ Adam) on BASELINE.json config 2 (8 keyframes at 640x480, N=500k, d=32, K=256, D=512) by
default; one "step" = one Stage-I iteration over the whole keyframe window
(total_objective + step_map + step_dict, proj/src/pipeline.cpp:236-246).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

N>1 runs under torchrun: the 8 keyframes are split across ranks (strong scaling), each rank
renders / decodes / back-propagates its frames, the gradient and loss buffers are summed with
NCCL all-reduce and every rank applies the same fused Adam. The time is the max over ranks.
``--impl reference`` times the reference's CPU algorithm (the C oracle port, all host threads)
on bounded row-band samples of the same workload and extrapolates to the full step.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "latent-map opt iters/s (render+dict-attn+bwd) 640x480, % roofline, vs CPU"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p["bf16_tflops_sustained"], "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic():
    """Per-launch DRAM bytes of each phase's kernels from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.py), or {} when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            k = json.load(f)["kernels"]
    except Exception:
        return {}
    out = {}
    for v in k.values():
        if v.get("phase"):
            out[v["phase"]] = out.get(v["phase"], 0.0) + v["bytes_per_launch"]
    return out


def ncu_warp_instructions():
    """Executed warp instructions per launch of each phase's kernels (same capture), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            k = json.load(f)["kernels"]
    except Exception:
        return {}
    out = {}
    for v in k.values():
        if v.get("phase") and v.get("warp_instructions_per_launch"):
            out[v["phase"]] = out.get(v["phase"], 0.0) + v["warp_instructions_per_launch"]
    return out


# ----------------------------------------------------------------------------- workload
def gpu_render_fn(ctx):
    import torch

    from paper_2602_12314_b200 import api

    def fn(m, q, t, intr):
        gm = api.GaussianMap.from_numpy(m)
        out = api.render(ctx, gm, api.make_pose(q, t),
                         api.make_intrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
        res = out.color.cpu().numpy(), out.depth.cpu().numpy(), out.alpha.cpu().numpy()
        del out, gm
        torch.cuda.synchronize()
        return res

    return fn


def decoder_flops_executed(n, k, ds, n_set):
    """Tensor-core flops the bf16 decoder kernels execute per frame (factored algebra)."""
    if k in (128, 256) and ds == 32 and n_set <= 64:
        # fused DEC1/DEC2: S = Q Kd^T, t = e M, dQ = dS Kd, R^T = dS^T Q; A = e^T (a e), Bm (64 columns)
        return 2.0 * n * k * (3 * ds + 2 * k + 64)
    # staged DL1-DL4: S twice, T = e M, dQ, R^T; gram over the upper-triangle units of A + Bm
    npx_t = -(-n // 128) * 128
    nb = max(16, -(-n_set // 16) * 16)
    nchunks = -(-(k + nb) // 256)
    gram = 0.0
    for mb in range(k // 128):
        for nc in range(mb // 2, nchunks):
            gram += 2.0 * 128 * min(256, k + nb - nc * 256) * npx_t
    return 2.0 * npx_t * k * (4 * ds + k) + gram


def decoder_flops_algorithmic(n, k, ds, df):
    return 6.0 * n * k * (ds + df)


def raster_bytes(n, v, pt, h, w, ds):
    """Algorithmic bytes per frame by kernel (SURVEY.md §8(d) formula, split per kernel)."""
    px = h * w
    return {
        "bin": n * 44 + n * 48 + pt * 8 * 2 * 2,
        "raster_fwd": pt * (48 + 12 + 4 * ds) + px * 4 * (5 + ds) + px * 8,
        "raster_bwd": pt * (48 + 12 + 4 * ds) + px * 4 * (4 + ds) + px * 8 + v * 4 * (10 + ds),
        "project_bwd": v * (44 + 48 + 32) + n * 4 * (14 + ds) * 0 + v * 4 * 12 * 2,
    }


# ----------------------------------------------------------------------------- reference arm
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference(cfg_id, samples, budget_s=150.0, threads=None, full_frame=False):
    """The reference's own CPU implementation (oracle/_ref: /root/reference/proj/src compiled with
    its Release flags against the Eigen stand-in; see oracle/ref/Makefile), timed on this host on
    row-band samples of one keyframe: t_objective(h) = a + b h is fitted over band heights and
    extrapolated to the full step, t_step = F (a + b H) + t_adam (Adam measured as a step minus an
    objective on the smallest band). Falls back to the C restatement when oracle/_ref is absent.
    ``full_frame`` additionally times one whole keyframe objective to check the band model."""
    from oracle import ref

    if not ref.available():
        return cpu_reference_port(cfg_id, samples, budget_s, threads)
    import oracle
    from paper_2602_12314_b200 import synthetic

    threads = threads or os.cpu_count() or 1
    oracle.set_gemm_threads(threads)

    def orender(m, q, t, intr):  # target images only (bit-identical to the reference's render)
        om = oracle.GaussianMap(*[np.ascontiguousarray(getattr(m, f), np.float32) for f in oracle.FIELDS])
        out = oracle.render(om, q, t, oracle.make_intr(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height),
                            threads=threads)
        return out["color"], out["depth"], out["alpha"]

    w = synthetic.make_workload(cfg_id, orender)
    W, H = w.intr.width, w.intr.height
    rcfg = ref.make_config(num_threads=threads, lambda_l2=w.lambdas["lambda_l2"], lambda_i2=w.lambdas["lambda_i2"],
                           lambda_trust=w.lambdas["lambda_trust"])
    heights = (16, 64) if H >= 128 else (2, 4)

    def band(fr, hb, pos):
        # the whole keyframe (full render, losses and backward), supervision kept on hb rows only:
        # the decoder's cost is linear in supervised rows, the rest is measured directly
        y0 = min(max(0, int(H * (pos + 0.5) / 4) - hb // 2), H - hb)
        asg = np.full_like(fr.assignment, -1)
        asg[y0:y0 + hb] = fr.assignment[y0:y0 + hb]
        return synthetic.Frame(fr.pose_rot, fr.pose_trans, fr.rgb, fr.depth, asg, fr.features), w.intr

    rows, t_obj = [], []
    t_start = time.time()
    t_adam = None
    for i in range(max(2, samples)):
        hb = heights[i % 2]
        f, intr = band(w.frames[i % len(w.frames)], hb, (i // 2) % 4)
        sess = ref.Session(w.map, w.atoms, w.anchor, w.proj, w.temperature, [f], intr, rcfg, threads)
        t0 = time.perf_counter()
        sess.objective()
        t1 = time.perf_counter()
        rows.append(hb)
        t_obj.append(t1 - t0)
        if t_adam is None and hb == heights[0]:
            t2 = time.perf_counter()
            sess.step()  # objective + MapOptimizer::step_map + step_dict
            t_adam = max(0.0, (time.perf_counter() - t2) - (t1 - t0))
        del sess
        if i >= 3 and time.time() - t_start > budget_s:
            break
    A = np.stack([np.ones(len(rows)), np.asarray(rows, np.float64)], 1)
    a, b = np.linalg.lstsq(A, np.asarray(t_obj), rcond=None)[0]
    a = max(a, 0.0)
    t_frame = a + b * H
    t_step = len(w.frames) * t_frame + (t_adam or 0.0)
    out = {
        "value": 1.0 / t_step, "unit": "iters/s", "cores": threads, "kind": "reference",
        "cpu_model": cpu_model(), "nproc": os.cpu_count(),
        "sample": (f"the reference itself (oracle/_ref: proj/src -O3 -DNDEBUG, no -march, Eigen stand-in with a "
                   f"single-threaded blocked SSE2 GEMM; num_threads={threads} for its parallel_chunks) on "
                   f"{len(rows)} full keyframes (render, losses, backward over all {W}x{H} px, N={w.map.n}) supervised on "
                   f"{heights[0]}/{heights[1]}-row bands at 4 heights; t_frame = a + b*supervised_rows fitted (the "
                   f"decoder is linear in rows), extrapolated to {H} rows x "
                   f"{len(w.frames)} frames + one Adam step (extrapolated); t_step={t_step:.1f}s, a={a:.3f}s, "
                   f"b={b:.4f}s/row, t_adam={t_adam or 0.0:.3f}s"),
        "seconds_spent": time.time() - t_start,
    }
    if full_frame:
        sess = ref.Session(w.map, w.atoms, w.anchor, w.proj, w.temperature, [w.frames[0]], w.intr, rcfg, threads)
        t0 = time.perf_counter()
        sess.objective()
        t_full = time.perf_counter() - t0
        out["full_keyframe"] = {"measured_s": t_full, "band_model_s": t_frame, "model_error": t_frame / t_full - 1.0}
    return out


def cpu_reference_port(cfg_id, samples, budget_s=150.0, threads=None):
    """Times the reference CPU algorithm (oracle port) on row-band samples of one keyframe and
    extrapolates linearly in band height: t_frame(h) = a + b h  ->  t_step = F (a + b H) + t_adam."""
    import oracle
    from paper_2602_12314_b200 import synthetic

    threads = threads or os.cpu_count() or 1
    oracle.build()

    def orender(m, q, t, intr):
        om = oracle.GaussianMap(*[np.ascontiguousarray(getattr(m, f), np.float32) for f in oracle.FIELDS])
        out = oracle.render(om, q, t, oracle.make_intr(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height),
                            threads=threads)
        return out["color"], out["depth"], out["alpha"]

    w = synthetic.make_workload(cfg_id, orender)
    W, H = w.intr.width, w.intr.height
    om = oracle.GaussianMap(*[np.ascontiguousarray(getattr(w.map, f), np.float32) for f in oracle.FIELDS])
    d = oracle.Dictionary(w.atoms.copy(), w.anchor.copy(), w.proj.copy(), np.float32(w.temperature))
    cfg = oracle.Config(lambda_l2=w.lambdas["lambda_l2"], lambda_i2=w.lambdas["lambda_i2"],
                        lambda_trust=w.lambdas["lambda_trust"])
    opt = oracle.MapOptimizer()
    heights = (4, 8) if H >= 64 else (2, 4)
    rows, t_obj, t_adam = [], [], []
    t_start = time.time()
    for i in range(max(2, samples)):
        hb = heights[i % 2]
        fr = w.frames[i % len(w.frames)]
        y0 = H // 2 - hb // 2
        intr = oracle.make_intr(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy - y0, W, hb)
        band = oracle.Frame(fr.pose_rot, fr.pose_trans, np.ascontiguousarray(fr.rgb[y0:y0 + hb]),
                            np.ascontiguousarray(fr.depth[y0:y0 + hb]),
                            np.ascontiguousarray(fr.assignment[y0:y0 + hb].reshape(-1)), fr.features)
        t0 = time.perf_counter()
        _, (g, dp, da) = oracle.total_objective(om, d, [band], intr, cfg, threads=threads)
        t1 = time.perf_counter()
        opt.step_map(om, g, cfg)
        opt.step_dict(d, dp, da, cfg)
        t2 = time.perf_counter()
        rows.append(hb)
        t_obj.append(t1 - t0)
        t_adam.append(t2 - t1)
        if i >= 1 and time.time() - t_start > budget_s:
            break
    A = np.stack([np.ones(len(rows)), np.asarray(rows, np.float64)], 1)
    a, b = np.linalg.lstsq(A, np.asarray(t_obj), rcond=None)[0]
    a = max(a, 0.0)
    t_frame = a + b * H
    t_step = len(w.frames) * t_frame + float(np.median(t_adam))
    return {
        "value": 1.0 / t_step, "unit": "iters/s", "cores": threads, "kind": "port", "cpu_model": cpu_model(),
        "sample": (f"oracle C port (reference algorithm, -O3, no -march) on {len(rows)} row-band samples "
                   f"({heights[0]}/{heights[1]} rows x {W} px of one keyframe, full N={w.map.n} projection), "
                   f"t_frame = a + b*rows fitted and extrapolated to {H} rows x {len(w.frames)} frames + Adam "
                   f"(extrapolated); t_step={t_step:.1f}s, a={a:.3f}s, b={b:.3f}s/row"),
        "seconds_spent": time.time() - t_start,
    }


# ----------------------------------------------------------------------------- config 3
def host_link_gbps(nbytes=256 << 20, reps=5):
    """Pinned cudaMemcpyAsync bandwidth H2D / D2H on this box (the PCIe roofline of the store's
    record transfers)."""
    import torch

    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    out = {}
    for name, dst, src in (("h2d", d, h), ("d2h", h, d)):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        out[name] = reps * nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9
    return out


def streaming_hash_pass(store, st, stats, sync_ms, hbm_peak):
    """The store's share of a config-3 frame (SURVEY.md §8(d) "Hash pass (K11)"): the device
    radius scan over every stored position against HBM, and the record traffic of sync (184 B per
    record written back or fetched) against the measured host link. Measured after the timed
    region."""
    import torch

    rec_bytes = 4 * (14 + 32)
    n = store.size()
    c = np.asarray(st.poses[-1][1], np.float32)
    store.fetch_local(c, st.radius)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        store.fetch_local(c, st.radius)
    scan_ms_host = (time.perf_counter() - t0) * 1000.0 / 5
    # the device radius scan (count + scan + emit into device scratch, one count readback)
    store.fetch_local_device(c, st.radius)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()  # the context's (and so the store's) stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    scan = []
    for _ in range(20):
        ev[0].record(stream)
        store.radius_scan(c, st.radius)  # count + scan + emit into device memory, no readback
        ev[1].record(stream)
        torch.cuda.synchronize()
        scan.append(ev[0].elapsed_time(ev[1]))
    scan_ms = float(np.median(scan))
    moved = [x["written_back"] + x["newborn_inserted"] + x["fetched"] for x in stats[-len(sync_ms):]]
    link = host_link_gbps()
    per_frame = float(np.mean(moved)) * rec_bytes if moved else 0.0
    sync_mean = float(np.mean(sync_ms)) if sync_ms else 0.0
    return {"records_scanned": n, "scan_bytes": 12 * n,
            "fetch_local_ms": scan_ms,
            "scan_gbps": 12 * n / (scan_ms * 1e-3) / 1e9,
            "scan_frac_hbm": 12 * n / (scan_ms * 1e-3) / 1e9 / hbm_peak,
            "scan_note": "device time of fetch_local's radius scan, CUDA events on the store's stream (radius count, "
                         "block scan, order-preserving emit into device memory; the count stays on the device); "
                         "median of 20; 12 B of position per stored record (count and emit both read them)",
            "fetch_local_host_ms": scan_ms_host,
            "record_bytes_per_frame": per_frame, "sync_ms_per_frame": sync_mean,
            "sync_share_of_frame": None,
            "transfer_gbps": per_frame / (sync_mean * 1e-3) / 1e9 if sync_mean else None,
            "transfer_note": "sync_ms covers the sync call; the written-back rows reach the pinned pool over PCIe "
                             "afterwards on the store's writeback stream, overlapping the frame's iterations",
            "host_link_gbps": link}


def run_streaming(args, hbm_peak):
    """Config 3: per frame one store sync (writeback of the optimised active set into the pinned
    host pool, prune by radius, fetch the newly active records; active_set.cpp:38-128) then 10
    Stage-I iterations on the frame. value = optimisation iterations/s over the timed frames
    (sync included); frames/s and the sync statistics are reported alongside."""
    import torch

    from paper_2602_12314_b200 import api, synthetic

    torch.cuda.set_device(0)
    ctx = api.Context(0)
    nfr = args.steps + args.warmup
    t0 = time.time()
    st = synthetic.make_streaming(nframes=nfr, device="cuda")
    intr = api.make_intrinsics(st.intr.fx, st.intr.fy, st.intr.cx, st.intr.cy, st.intr.width, st.intr.height)
    store = api.Store(ctx, st.capacity, 32)
    inserted = store.insert_global(st.records, st.voxel_size)
    del st.records
    # targets: a perturbed copy of each frame's active set rendered on the device (as configs 0-2)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(synthetic.seed_for(3))
    frames = []
    for f, (q, t) in enumerate(st.poses):
        _, rec = store.fetch_local(np.asarray(t, np.float32), st.radius, gather=True)
        pos = rec[:, 0:3] + 0.01 * torch.randn(rec[:, 0:3].shape, generator=gen, device="cuda")
        col = (rec[:, 7:10] + 0.05 * torch.randn(rec[:, 7:10].shape, generator=gen, device="cuda")).clamp(0, 1)
        gm = api.GaussianMap(pos.contiguous(), rec[:, 3:7].contiguous(), col.contiguous(), rec[:, 10:13].contiguous(),
                             rec[:, 13].contiguous(), rec[:, 14:].contiguous())
        out = api.render(ctx, gm, api.make_pose(q, t), intr)
        alpha = out.alpha
        depth = torch.where(alpha > 0.5, out.depth, torch.zeros_like(out.depth))
        frames.append(synthetic.Frame(q, t, *[torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy() for a in (
            out.color.cpu().numpy(), depth.cpu().numpy(), st.assignments[f], st.features[f])]))
        del out, gm, rec
    gen_s = time.time() - t0
    cfg = api.default_config(**st.lambdas)
    cfg.decoder_precision = 1
    s = api.Session(ctx, cfg, 0, 32, st.atoms.shape[0], st.atoms.shape[1], intr)
    s.set_dictionary(st.atoms, st.atoms, st.proj)
    origin = torch.zeros(0, dtype=torch.int64, device="cuda")
    stats_all, active, vis_all, pairs_all, sync_ms = [], [], [], [], []

    def one_frame(f):
        nonlocal origin
        q, t = st.poses[f]
        ts = time.perf_counter()
        rows = s.export_rows() if s.n else None
        # device-resident sync: every row dirty after Stage I (d_dirty = None), origins / kept mask
        # stay on the device, the counts come back once
        d_out, origin_new, kept, stats = store.sync_device(rows, origin, None, np.asarray(t, np.float32), st.radius,
                                                           st.voxel_size)
        n_kept = int(d_out.shape[0]) - stats["fetched"]
        s.import_rows_device(d_out, kept if origin.numel() else None, n_kept if origin.numel() else 0)
        sync_ms.append((time.perf_counter() - ts) * 1000.0)  # host clock around export + sync + import
        origin = origin_new.clone()
        s.set_frames([frames[f]])
        s.set_batch(1)
        for _ in range(st.iters_per_frame):
            s.step(read=False)
        return stats

    for f in range(args.warmup):
        one_frame(f)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    sampler = ClockSampler(0)
    sampler.start()
    launches0 = ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tw = time.perf_counter()
    ev0.record(stream)
    for f in range(args.warmup, nfr):
        stats_all.append(one_frame(f))
        active.append(s.n)
        vis_f, pairs_f = s.stats(1)
        vis_all.append(float(vis_f[0]))
        pairs_all.append(float(pairs_f[0]))
    ev1.record(stream)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - tw) * 1000.0
    ms = max(ev0.elapsed_time(ev1), wall)
    clocks = sampler.stop()
    last = s.read_loss()
    iters = args.steps * st.iters_per_frame
    moved = sum(x["fetched"] + x["written_back"] for x in stats_all)
    hash_pass = streaming_hash_pass(store, st, stats_all, sync_ms[args.warmup:], hbm_peak)
    hash_pass["sync_share_of_frame"] = sum(sync_ms[args.warmup:]) / ms if ms else None
    line = {"metric": METRIC, "value": 1000.0 * iters / ms, "unit": "iters/s", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "replicas only",
            "vs_baseline": None, "dtype": "f32 render/grads, bf16 tcgen05 decoder (fp32 accum)",
            "data": "synthetic (seeded BASELINE config 3; targets rendered from a perturbed active set)",
            "config": {"workload": st.name, "frames_timed": args.steps, "iters_per_frame": st.iters_per_frame,
                       "image": f"{st.intr.width}x{st.intr.height}", "global_records": int(inserted),
                       "voxel_size_m": st.voxel_size, "hash_capacity": st.capacity, "radius_m": st.radius,
                       "query_dim": 32, "dict_K": 256, "embed_D": 1024, "parallelism": "single GPU",
                       "step": "one step = one frame: store sync + 10 Stage-I iterations"},
            "frames_per_s": 1000.0 * args.steps / ms, "active_mean": float(np.mean(active)),
            "visible_per_frame": float(np.mean(vis_all)), "tile_pairs_per_frame": float(np.mean(pairs_all)),
            "records_moved_per_frame": moved / max(1, args.steps),
            "sync_stats_last": stats_all[-1] if stats_all else None, "hash_pass": hash_pass,
            "gpu_launches": int(ctx.launches() - launches0),
            "clocks": clocks, "loss_last": last["total"], "setup_s": gen_s}
    print(json.dumps(line))


# ----------------------------------------------------------------------------- launch
def relaunch(args):
    """`bench.py --gpus N` started as one process: re-exec under torch.distributed.run with one
    rank per GPU (127.0.0.1 rendezvous), NCCL's INFO lines on stderr. N is capped at the visible
    GPU count; the JSON line's n_gpus is the number of ranks that actually ran."""
    import socket

    import torch

    avail = torch.cuda.device_count()
    n = min(args.gpus, avail) if avail > 0 else 1
    if n < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested, {avail} visible: running {n} rank(s)", file=sys.stderr)
    argv = [a for a in sys.argv[1:]]
    if n == 1:
        os.environ["WORLD_SIZE"] = "1"
        return main()
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + argv
    rc = subprocess.call(cmd, env=env)
    if rc != 0:
        sys.exit(rc)


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--exchange", default="sharded", choices=["sharded", "allreduce"],
                    help="N>1: ZeRO-1 sharded Adam (default) or all-reduce + replicated Adam")
    ap.add_argument("--cpu-full-frame", action="store_true",
                    help="reference arm: also time one whole keyframe to check the row-band model")
    ap.add_argument("--profile-phases", type=int, default=1)
    ap.add_argument("--decoder-path", type=int, default=0,
                    help="bf16 decoder kernels: 0 auto, 1 fused on-chip, 2 staged (experiments)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        return relaunch(args)
    if args.config == 3 and args.impl == "ours":
        return run_streaming(args, peaks()[0])
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2602_12314_b200 import synthetic

    cfg_name = synthetic.NAMES[args.config]
    config = {"workload": cfg_name, "keyframes": synthetic.SPECS[args.config][-1],
              "gaussians": synthetic.SPECS[args.config][5], "query_dim": synthetic.SPECS[args.config][8],
              "dict_K": synthetic.SPECS[args.config][9], "embed_D": synthetic.SPECS[args.config][10],
              "image": f"{synthetic.SPECS[args.config][0]}x{synthetic.SPECS[args.config][1]}",
              "parallelism": f"keyframe-sharded x{world}" if world > 1 else "single GPU",
              "l2": "working set > L2 (126 MB) every step; no explicit flush",
              "launch": "each Stage-I step replayed as one captured CUDA graph (N=1)",
              "streams": "renders of all keyframes ahead on a render stream; frame b's render backward on a "
                         "backward stream overlapping frame b+1's losses + decoder; joined inside the graph",
              "phases_note": "per-phase times are measured single-stream (phase profiling disables the overlap)"}

    if args.impl == "reference":
        if rank != 0:
            return
        ref = cpu_reference(args.config, args.steps + args.warmup, full_frame=args.cpu_full_frame)
        line = {"impl": "reference", "metric": METRIC, "value": ref["value"], "unit": "iters/s",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1000.0 / ref["value"], "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE config)",
                "config": config, "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")},
                "full_keyframe_check": ref.get("full_keyframe"),
                "e2e": {"value": ref["value"], "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch

    from paper_2602_12314_b200 import api

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    ctx = api.Context(local_rank)
    ctx.set_decoder_path(args.decoder_path)
    w = synthetic.make_workload(args.config, gpu_render_fn(ctx))
    from paper_2602_12314_b200.sharding import rank_plan

    nf = len(w.frames)
    plan = rank_plan(nf, world, rank)
    mine = [w.frames[i] for i in plan["frames"]]
    cfg = api.default_config(**w.lambdas)
    # BASELINE: config 0 is all fp32; configs 1-4 decode in bf16 with fp32 accumulation (tcgen05)
    cfg.decoder_precision = 0 if args.config == 0 else 1
    intr = api.make_intrinsics(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height)
    s = api.Session(ctx, cfg, w.map.n, w.map.features.shape[1], w.atoms.shape[0], w.atoms.shape[1], intr)
    s.set_map(w.map)
    s.set_dictionary(w.atoms, w.anchor, w.proj)
    # pinned host copies of this rank's keyframes (the e2e path copies them H2D every step)
    pinned = []
    for f in mine:
        pf = synthetic.Frame(f.pose_rot, f.pose_trans,
                             *[torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
                               for a in (f.rgb, f.depth, f.assignment, f.features)])
        pinned.append(pf)
    s.set_frames(pinned)
    s.set_batch(plan["global_batch"], add_trust=plan["add_trust"], slot_offset=plan["slot_offset"])
    grads = s.grad_buffer()
    parts = s.loss_buffer()
    comm, collective = None, None
    if world > 1:
        # the exchange through the library's own NCCL communicator (latmap_session_allreduce);
        # torch.distributed's all-reduce of the same buffers if NCCL cannot be loaded there
        try:
            uid = [api.Comm.unique_id(ctx) if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            comm = api.Comm(ctx, world, rank, uid[0])
            collective = "latmap_session_allreduce (NCCL sum, one group)"
        except Exception as e:  # noqa: BLE001
            comm, collective = None, f"torch.distributed.all_reduce (library comm unavailable: {e})"
        config["collective"] = collective

    sharded_adam = args.exchange == "sharded" and comm is not None
    if world > 1:
        config["exchange"] = ("ZeRO-1: reduce-scatter grads, shard check, all-reduce loss partials, Adam on the "
                              "rank's shard, all-gather params (latmap_session_exchange_sharded)" if sharded_adam
                              else "all-reduce grads + loss partials, replicated Adam")

    def exchange(sess):
        if sharded_adam:
            comm.session_exchange_sharded(sess)
        elif comm is not None:
            comm.session_allreduce(sess)
        else:
            dist.all_reduce(grads)
            dist.all_reduce(parts)

    def one_step(read=False):
        if world == 1:
            return s.step(read=read)
        return s.sharded_step(exchange, read=read, apply=not sharded_adam)

    stream = torch.cuda.current_stream()
    first = one_step(read=True)  # sizes the tile buffers
    for _ in range(max(0, args.warmup - 1)):
        one_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.25)
    launches0 = ctx.launches()
    overflow0 = s.overflow_steps()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        one_step()
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launches() - launches0
    # sticky device count of steps whose Adam was skipped for a tile-list overflow (any rank) during
    # the timed loop, which reads no losses: 0 means every timed step was whole
    overflowed = s.overflow_steps() - overflow0
    clocks = sampler.stop()
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = 1000.0 / ms_per_step

    # e2e through the public API: H2D of the step's keyframes from pinned memory, the step,
    # D2H of the step's loss. On one GPU the loss partials of step k come back asynchronously
    # (pinned buffer) and are assembled while step k+1 runs -- a training loop's lagged loss read,
    # no per-step stall; with N ranks every step reads its LossBreakdown synchronously.
    h2d = sum(f.rgb.nbytes + f.depth.nbytes + f.assignment.nbytes + f.features.nbytes for f in pinned)
    d2h = 48
    lbuf = [torch.empty(4096, dtype=torch.float64).pin_memory().numpy() for _ in range(2)]
    lev = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e_steps = max(3, args.steps // 2)
    t0 = time.perf_counter()
    e0.record(stream)
    for k in range(e_steps):
        s.set_frames(pinned)
        if world == 1:
            one_step(read=False)
            nl = s.read_loss_async(lbuf[k % 2])
            lev[k % 2].record(stream)
            d2h = 8 * nl
            if k > 0:
                lev[(k - 1) % 2].synchronize()
                last = api.assemble_loss(lbuf[(k - 1) % 2][:nl], w.intr.width, w.intr.height, cfg)
        else:
            last = one_step(read=True)
    if world == 1:
        lev[(e_steps - 1) % 2].synchronize()
        last = api.assemble_loss(lbuf[(e_steps - 1) % 2][:nl], w.intr.width, w.intr.height, cfg)
    e1.record(stream)
    torch.cuda.synchronize()
    e_wall = (time.perf_counter() - t0) * 1000.0
    e_ms = max(e0.elapsed_time(e1), e_wall)
    if dist:
        t = torch.tensor([e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t.item())
    e2e = {"value": 1000.0 * e_steps / e_ms, "unit": "iters/s", "h2d_bytes_per_step": int(h2d) * world,
           "d2h_bytes_per_step": d2h * world, "steps": e_steps,
           "note": "timed after the device-resident loop, on later steps of the same optimisation: the map "
                   "moves every step and the tile-pair count (the work) drifts by a few percent, so e2e and "
                   "value can differ either way by that much"}

    # phase breakdown (CUDA events per phase; steps run uncaptured while profiling), after the timed
    # region so the events do not perturb it
    phases = {}
    if args.profile_phases:
        torch.cuda.synchronize()
        s.profile(True)
        s.phase_times()
        for _ in range(3):
            one_step()
        torch.cuda.synchronize()
        phases = s.phase_times()
        s.profile(False)
    # roofline of the dominant kernel (phase), per launch
    hbm, bf16_burst, bf16_sus, src = peaks()
    vis, pairs = s.stats(len(mine))
    H, W = w.intr.height, w.intr.width
    n, ds, K, D = w.map.n, w.map.features.shape[1], w.atoms.shape[0], w.atoms.shape[1]
    per_launch = {}
    for ph, (tms, cnt) in phases.items():
        if cnt == 0:
            continue
        per_launch[ph] = {"ms_per_launch": tms / cnt, "launches": cnt, "share": None}
    total_ph = sum(v[0] for v in phases.values()) or 1.0
    for ph in per_launch:
        per_launch[ph]["share"] = phases[ph][0] / total_ph
    rb = raster_bytes(n, float(np.mean(vis)), float(np.mean(pairs)), H, W, ds)
    traffic = ncu_traffic()
    roof = None
    if per_launch:
        dom = max(per_launch, key=lambda p: phases[p][0])
        t_launch = per_launch[dom]["ms_per_launch"] / 1000.0
        if dom == "decoder":
            n_set = max(int(f.features.shape[0]) for f in w.frames)
            fe = decoder_flops_executed(H * W, K, ds, n_set)
            fa = decoder_flops_algorithmic(H * W, K, ds, D)
            # achieved = SURVEY.md §8(d) algorithmic flops 6 n K (d_s + d_f) per frame / time; the
            # factored algebra executes fewer (executed_* fields), never reported above peak
            roof = {"kernel": "decoder (fused feature loss + backward, factored algebra)", "bound": "tensor",
                    "achieved": fa / t_launch / 1e12, "peak": bf16_sus, "unit": "TFLOP/s",
                    "frac": min(1.0, fa / t_launch / 1e12 / bf16_sus), "traffic": traffic.get("decoder"),
                    "algorithmic_per_launch": fa, "peak_source": f"{src} bf16 sustained",
                    "executed_per_launch": fe, "executed_tflops": fe / t_launch / 1e12,
                    "executed_frac": fe / t_launch / 1e12 / bf16_sus}
        elif dom in rb:
            by = rb[dom]
            roof = {"kernel": dom, "bound": "hbm", "achieved": by / t_launch / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": by / t_launch / 1e9 / hbm, "traffic": traffic.get(dom), "algorithmic_per_launch": by,
                    "peak_source": f"{src} HBM copy"}
            wi = ncu_warp_instructions().get(dom) if args.config == 2 else None
            if wi:  # the rasteriser is issue-bound: its instruction issue rate against the SMs' peak
                clk = (clocks or {}).get("sm_mhz") or 1965.0
                peak_i = 148 * 4 * clk * 1e6  # one warp instruction per scheduler per clock
                roof["issue"] = {"warp_instructions_per_launch": wi, "achieved": wi / t_launch, "peak": peak_i,
                                 "unit": "warp instructions/s", "frac": wi / t_launch / peak_i,
                                 "source": "smsp__inst_executed.sum of the committed ncu --set full capture "
                                           "(profiles/ncu_traffic.json); time per launch measured live"}
        else:
            roof = {"kernel": dom, "bound": "hbm", "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None,
                    "traffic": None}
    line = {"metric": METRIC, "value": value * 1.0, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32" if cfg.decoder_precision == 0 else "f32 render/grads, bf16 tcgen05 decoder (fp32 accum)",
            "data": "synthetic (seeded BASELINE config; targets rendered from a perturbed map)",
            "config": config, "roofline": roof, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
            "overflowed_steps": int(overflowed),
            "phases": {k: round(v["ms_per_launch"], 4) for k, v in per_launch.items()},
            "phase_share": {k: round(v["share"], 4) for k, v in per_launch.items()},
            "visible_per_frame": float(np.mean(vis)), "tile_pairs_per_frame": float(np.mean(pairs)),
            "loss_first": first["total"] if first else None, "loss_last": last["total"] if last else None}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ref = cpu_reference(args.config, 6, budget_s=40.0)
        line["cpu_baseline"] = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
