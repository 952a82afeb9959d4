"""Python mirror of the reference operator API (proj/include/latmap/**) over the C-ABI.

Same names, argument meaning and error behaviour as the reference:
``render`` / ``render_backward`` (splat/render.hpp:97-119), ``reconstruct`` /
``reconstruct_backward`` / ``trust_region_penalty`` (dict/dictionary.hpp:63-77),
``ssim`` (obj/losses.hpp:12-13), ``adam_step`` (obj/adam.hpp:61-79) and the
device-resident ``Session`` running Stage-I iterations (total_objective +
MapOptimizer::step_map/step_dict, objective.cpp:67-194 / pipeline.cpp:75-95).
Tensors are torch CUDA float32 (torch is only the device-memory plumbing).
"""
from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, fields

import numpy as np
import torch

from . import _capi
from ._capi import Config, Frame, Intrinsics, LossBreakdown, MapView, Pose, check, lib

MAP_FIELDS = ("positions", "rotations", "colors", "log_scales", "opacity_logits", "features")


def _ptr(t):
    if t is None:
        return None
    assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous(), "expected contiguous cuda float32"
    return C.c_void_p(t.data_ptr())


def _iptr(t, dtype=torch.int32):
    """Device pointer of a contiguous CUDA integer tensor."""
    assert t.is_cuda and t.dtype == dtype and t.is_contiguous(), f"expected contiguous cuda {dtype}"
    return C.c_void_p(t.data_ptr())


@dataclass
class GaussianMap:
    """GaussianMapT<float> on the device (core/types.hpp:93-199)."""
    positions: torch.Tensor
    rotations: torch.Tensor
    colors: torch.Tensor
    log_scales: torch.Tensor
    opacity_logits: torch.Tensor
    features: torch.Tensor

    @property
    def n(self):
        return self.positions.shape[0]

    @property
    def query_dim(self):
        return self.features.shape[1]

    def view(self):
        return MapView(self.n, self.query_dim, *[_ptr(getattr(self, f)) for f in MAP_FIELDS])

    @staticmethod
    def from_numpy(m, device="cuda"):
        return GaussianMap(*[torch.as_tensor(np.ascontiguousarray(getattr(m, f), np.float32), device=device)
                             for f in MAP_FIELDS])

    def zeros_like(self):
        return GaussianMap(*[torch.zeros_like(getattr(self, f)) for f in MAP_FIELDS])

    def numpy(self):
        return {f: getattr(self, f).detach().cpu().numpy() for f in MAP_FIELDS}


def make_pose(rotation=(1, 0, 0, 0), translation=(0, 0, 0)):
    return Pose((C.c_float * 4)(*[float(v) for v in rotation]), (C.c_float * 3)(*[float(v) for v in translation]))


def make_intrinsics(fx, fy, cx, cy, width, height):
    return Intrinsics(fx, fy, cx, cy, width, height)


_UNIFORM = C.CFUNCTYPE(C.c_double, C.c_void_p)


def _uniform_arg(uniform):
    """(fn, user, keepalive) for a latmap_uniform_fn argument."""
    if callable(uniform):
        cb = _UNIFORM(lambda _user: float(uniform()))
        return C.cast(cb, C.c_void_p), None, cb
    fn, user = uniform
    return C.c_void_p(fn), C.c_void_p(user), None


class Context:
    """A latmap_ctx bound to one device and torch's current stream."""

    def __init__(self, device=0):
        self.device = device
        torch.cuda.set_device(device)
        self.stream = torch.cuda.current_stream(device)
        h = C.c_void_p()
        st = lib().latmap_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h))
        check(None, st)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().latmap_ctx_destroy(self.h)
            except TypeError:  # interpreter shutdown: the library handle is already gone
                pass
            self.h = None

    def sync(self):
        check(self.h, lib().latmap_ctx_synchronize(self.h))

    def set_exact_blend(self, exact=True):
        check(self.h, lib().latmap_ctx_set_exact_blend(self.h, int(bool(exact))))

    def set_deterministic(self, on=True):
        """Fixed-order gradient reductions: bit-identical gradients run to run (slower)."""
        check(self.h, lib().latmap_ctx_set_deterministic(self.h, int(bool(on))))

    def set_decoder_path(self, path):
        """bf16 decoder kernels: 0 auto, 1 fused on-chip (DEC1/DEC2), 2 staged (DL1-DL5)."""
        check(self.h, lib().latmap_ctx_set_decoder_path(self.h, int(path)))

    def set_reconstruct_precision(self, precision):
        """Standalone reconstruct / query_map / evaluation: 0 fp32, 1 bf16 tcgen05 (K in 256..1024,
        d_s in {32, 64}, D a multiple of 256; other shapes stay fp32)."""
        check(self.h, lib().latmap_ctx_set_reconstruct_precision(self.h, int(precision)))

    def weighted_kmeans(self, points, weights, k, uniform, warm=None, max_iters=10):
        """weighted_kmeans (stream_kmeans.cpp:94-157) on the device -> (centers, weights, iterations).

        ``uniform`` supplies std::uniform_real_distribution<double>(0, 1) draws of the caller's
        generator: a Python callable, or a (C function pointer, user pointer) pair."""
        pts = np.ascontiguousarray(points, np.float32)
        w = np.ascontiguousarray(weights, np.float32)
        n, dim = pts.shape
        cen = np.zeros((k, dim), np.float32)
        cw = np.zeros(k, np.float32)
        it = C.c_int32(0)
        wm = None if warm is None else np.ascontiguousarray(warm, np.float32)
        fn, user, keep = _uniform_arg(uniform)
        check(self.h, lib().latmap_weighted_kmeans(
            self.h, pts.ctypes.data_as(C.c_void_p), w.ctypes.data_as(C.c_void_p), n, dim, int(k), fn, user,
            None if wm is None else wm.ctypes.data_as(C.c_void_p), 0 if wm is None else wm.shape[0], int(max_iters),
            cen.ctypes.data_as(C.c_void_p), cw.ctypes.data_as(C.c_void_p), C.byref(it)))
        del keep
        return cen, cw, it.value

    def launches(self):
        return lib().latmap_ctx_launch_count(self.h)


class RenderOutput:
    """RenderOutputT<float> (splat/render.hpp:41-53): images + the projection cache."""

    def __init__(self, ctx, color, depth, query, alpha, cache):
        self.ctx, self.color, self.depth, self.query, self.alpha, self._cache = ctx, color, depth, query, alpha, cache

    def __del__(self):
        if getattr(self, "_cache", None):
            try:
                lib().latmap_render_cache_destroy(self._cache)
            except TypeError:  # interpreter shutdown: the library handle is already gone
                pass
            self._cache = None

    def splats(self):
        """ProjectedSplat records of the surviving splats in source order (numpy structured)."""
        L = lib()
        cnt = C.c_int64(0)
        check(self.ctx.h, L.latmap_render_cache_splats(self.ctx.h, self._cache, None, 0, C.byref(cnt)))
        arr = (_capi.ProjectedSplat * max(cnt.value, 1))()
        check(self.ctx.h, L.latmap_render_cache_splats(self.ctx.h, self._cache, arr, cnt.value, C.byref(cnt)))
        dt = np.dtype([("mean", np.float32, 2), ("cov_inv", np.float32, 4), ("depth", np.float32),
                       ("alpha", np.float32), ("source", np.int32), ("x0", np.int32), ("x1", np.int32),
                       ("y0", np.int32), ("y1", np.int32)])
        return np.frombuffer(bytes(arr), dtype=dt, count=cnt.value).copy()

    def tiles(self):
        """(tiles_x, tiles_y, offsets[ntiles+1], sources[pairs]) of the canonical tile lists."""
        L = lib()
        tx, ty, pairs = C.c_int32(), C.c_int32(), C.c_int64()
        check(self.ctx.h, L.latmap_render_cache_tiles(self.ctx.h, self._cache, None, None, 0, C.byref(tx),
                                                      C.byref(ty), C.byref(pairs)))
        off = np.zeros(tx.value * ty.value + 1, np.int32)
        src = np.zeros(max(pairs.value, 1), np.int32)
        check(self.ctx.h, L.latmap_render_cache_tiles(self.ctx.h, self._cache, off.ctypes.data_as(C.c_void_p),
                                                      src.ctypes.data_as(C.c_void_p), pairs.value, None, None, None))
        return tx.value, ty.value, off, src[: pairs.value]


def project_gaussian(ctx, position, rotation, log_scale, opacity_logit, pose, intr):
    """project_gaussian (splat/render.hpp:97-99); None when culled."""
    arrs = [np.ascontiguousarray(a, np.float32) for a in (position, rotation, log_scale)]
    vis = C.c_int32(0)
    mean = np.zeros(2, np.float32)
    cov = np.zeros(4, np.float32)
    depth = np.zeros(1, np.float32)
    check(ctx.h, lib().latmap_project_gaussian(ctx.h, *[a.ctypes.data_as(C.c_void_p) for a in arrs],
                                               float(opacity_logit), C.byref(pose), C.byref(intr), C.byref(vis),
                                               mean.ctypes.data_as(C.c_void_p), cov.ctypes.data_as(C.c_void_p),
                                               depth.ctypes.data_as(C.c_void_p)))
    if not vis.value:
        return None
    return mean, cov.reshape(2, 2), float(depth[0])


def render(ctx, m: GaussianMap, pose, intr) -> RenderOutput:
    """render (splat/render.hpp:103-105)."""
    h, w = intr.height, intr.width
    dev = m.positions.device
    color = torch.empty((h, w, 3), device=dev)
    depth = torch.empty((h, w), device=dev)
    query = torch.empty((h, w, m.query_dim), device=dev)
    alpha = torch.empty((h, w), device=dev)
    cache = C.c_void_p()
    check(ctx.h, lib().latmap_render_cache_create(ctx.h, C.byref(cache)))
    out = RenderOutput(ctx, color, depth, query, alpha, cache)
    mv = m.view()
    check(ctx.h, lib().latmap_render(ctx.h, C.byref(mv), C.byref(pose), C.byref(intr), cache, _ptr(color),
                                     _ptr(depth), _ptr(query), _ptr(alpha)))
    return out


def render_backward(ctx, m: GaussianMap, pose, intr, out: RenderOutput, d_color=None, d_depth=None, d_query=None):
    """render_backward (splat/render.hpp:116-119) -> MapGradients (fresh zeros + accumulated)."""
    g = m.zeros_like()
    mv, gv = m.view(), g.view()
    check(ctx.h, lib().latmap_render_backward(ctx.h, C.byref(mv), C.byref(pose), C.byref(intr), out._cache,
                                              _ptr(d_color), _ptr(d_depth), _ptr(d_query), C.byref(gv)))
    return g


def reconstruct(ctx, queries, atoms, proj, temperature, want_attention=False):
    """reconstruct (dict/dictionary.hpp:63-65)."""
    n, ds = queries.shape
    k, df = atoms.shape
    if proj.shape[0] != ds:
        raise _capi.InvalidArgument("reconstruct: query dimension mismatch")
    if proj.shape[1] != df:
        raise _capi.InvalidArgument("reconstruct: projection/atom dimension mismatch")
    out = torch.empty((n, df), device=queries.device)
    att = torch.empty((n, k), device=queries.device) if want_attention else None
    check(ctx.h, lib().latmap_reconstruct(ctx.h, _ptr(queries), n, ds, _ptr(atoms), _ptr(proj), k, df,
                                          float(temperature), _ptr(out), _ptr(att)))
    return (out, att) if want_attention else out


def reconstruct_backward(ctx, queries, attention, atoms, proj, temperature, d_rec):
    """reconstruct_backward (dict/dictionary.hpp:67-70)."""
    n, ds = queries.shape
    k, df = atoms.shape
    dq = torch.empty_like(queries)
    dp = torch.empty_like(proj)
    da = torch.empty_like(atoms)
    check(ctx.h, lib().latmap_reconstruct_backward(ctx.h, _ptr(queries), _ptr(attention), n, ds, _ptr(atoms),
                                                   _ptr(proj), k, df, float(temperature), _ptr(d_rec), _ptr(dq),
                                                   _ptr(dp), _ptr(da)))
    return dict(d_queries=dq, d_proj=dp, d_atoms=da)


def trust_region_penalty(ctx, atoms, anchor, delta, want_grad=False):
    """trust_region_penalty (dict/dictionary.hpp:75-77)."""
    if atoms.shape != anchor.shape:
        raise _capi.InvalidArgument("trust_region_penalty: shape mismatch")
    g = torch.empty_like(atoms) if want_grad else None
    v = C.c_float(0)
    check(ctx.h, lib().latmap_trust_region_penalty(ctx.h, _ptr(atoms), _ptr(anchor), atoms.shape[0], atoms.shape[1],
                                                   float(delta), _ptr(g), C.byref(v)))
    return (v.value, g) if want_grad else v.value


def ssim(ctx, a, b, want_grad=False):
    """ssim (obj/losses.hpp:12-13) on HxWxC (or HxW) images."""
    if a.shape != b.shape:
        raise _capi.InvalidArgument("ssim: image shapes differ")
    h, w = a.shape[:2]
    ch = a.shape[2] if a.dim() == 3 else 1
    da = torch.empty_like(a) if want_grad else None
    v = C.c_float(0)
    check(ctx.h, lib().latmap_ssim(ctx.h, _ptr(a), _ptr(b), h, w, ch, _ptr(da), C.byref(v)))
    return (v.value, da) if want_grad else v.value


def rgb_loss(ctx, rendered, observed, lambda_i1, lambda_i2, want_grad=True):
    """rgb_loss (obj/losses.hpp:33-34): {value, l1, ssim_loss, grad} on HxWxC device images."""
    if rendered.shape != observed.shape:
        raise _capi.InvalidArgument("rgb_loss: image shapes differ")
    h, w = rendered.shape[:2]
    ch = rendered.shape[2] if rendered.dim() == 3 else 1
    g = torch.empty_like(rendered) if want_grad else None
    v, l1, ss = C.c_float(), C.c_float(), C.c_float()
    check(ctx.h, lib().latmap_rgb_loss(ctx.h, _ptr(rendered), _ptr(observed), h, w, ch, float(lambda_i1),
                                       float(lambda_i2), _ptr(g), C.byref(v), C.byref(l1), C.byref(ss)))
    return {"value": v.value, "l1": l1.value, "ssim_loss": ss.value, "grad": g}


def depth_loss(ctx, rendered, observed, alpha, want_grad=True):
    """depth_loss (obj/losses.hpp:38-40): {value, flagged, grad} on HxW device images."""
    if rendered.shape != observed.shape or rendered.shape != alpha.shape:
        raise _capi.InvalidArgument("depth_loss: image shapes differ")
    g = torch.empty_like(rendered) if want_grad else None
    v, fl = C.c_float(), C.c_int32()
    check(ctx.h, lib().latmap_depth_loss(ctx.h, _ptr(rendered), _ptr(observed), _ptr(alpha), rendered.numel(),
                                         _ptr(g), C.byref(v), C.byref(fl)))
    return {"value": v.value, "flagged": bool(fl.value), "grad": g}


def feature_loss(ctx, reconstructed, target, atoms, anchor, delta, lambda_cos, lambda_l2, lambda_trust,
                 want_grad=True):
    """feature_loss (obj/losses.hpp:43-58): {value, cos_term, l2_term, trust_term,
    zero_norm_flagged, d_reconstructed, d_atoms_trust} on device rows."""
    if reconstructed.shape != target.shape:
        raise _capi.InvalidArgument("feature_loss: shape mismatch")
    n, df = reconstructed.shape
    k = atoms.shape[0]
    dr = torch.empty_like(reconstructed) if want_grad else None
    dt = torch.empty_like(atoms) if want_grad else None
    terms = (C.c_float * 4)()
    fl = C.c_int32()
    check(ctx.h, lib().latmap_feature_loss(ctx.h, _ptr(reconstructed), _ptr(target), n, df, _ptr(atoms), _ptr(anchor),
                                           k, float(delta), float(lambda_cos), float(lambda_l2), float(lambda_trust),
                                           _ptr(dr), _ptr(dt), terms, C.byref(fl)))
    return {"value": terms[0], "cos_term": terms[1], "l2_term": terms[2], "trust_term": terms[3],
            "zero_norm_flagged": bool(fl.value), "d_reconstructed": dr, "d_atoms_trust": dt}


# --------------------------------------------------------------------------- evaluation
def gather_supervision(ctx, query, assignment, features, normalize=False):
    """gather_supervision, pixel mode (objective.cpp:16-35) on the device -> (queries n x ds,
    targets n x df, pixel_of_row n). ``normalize`` divides each target row by its norm (> 1e-12),
    as evaluate_map does (evaluate.cpp:38-42)."""
    q = query.reshape(-1, query.shape[-1]).contiguous()
    asg = assignment.reshape(-1).to(torch.int32).contiguous()
    feats = features.contiguous()
    npx, ds = q.shape
    df = feats.shape[1]
    n = C.c_int64(0)
    check(ctx.h, lib().latmap_gather_supervision(ctx.h, _ptr(q), ds, _iptr(asg), npx, _ptr(feats), df, int(normalize),
                                                 None, None, None, 0, C.byref(n)))
    qo = torch.empty((n.value, ds), device=q.device)
    to = torch.empty((n.value, df), device=q.device)
    po = torch.empty(n.value, dtype=torch.int64, device=q.device)
    check(ctx.h, lib().latmap_gather_supervision(ctx.h, _ptr(q), ds, _iptr(asg), npx, _ptr(feats), df, int(normalize),
                                                 _ptr(qo), _ptr(to), _iptr(po, torch.int64), n.value, C.byref(n)))
    return qo, to, po


def metric_cos(ctx, rec, tgt):
    """metric_cos (io/metrics.hpp:12-13) -> (value, flagged)."""
    if rec.shape != tgt.shape:
        raise _capi.InvalidArgument("metric_cos: shape mismatch")
    v, fl = C.c_double(0), C.c_int32(0)
    check(ctx.h, lib().latmap_metric_cos(ctx.h, _ptr(rec.contiguous()), _ptr(tgt.contiguous()), rec.shape[0],
                                         rec.shape[1], C.byref(v), C.byref(fl)))
    return v.value, bool(fl.value)


def metric_miou(ctx, emb, labels, prototypes):
    """metric_miou (io/metrics.hpp:15-26) -> (miou, intersection, union) (numpy int64 per class)."""
    lab = labels.to(torch.int32).contiguous()
    c = prototypes.shape[0]
    inter = np.zeros(c, np.int64)
    uni = np.zeros(c, np.int64)
    v = C.c_double(0)
    check(ctx.h, lib().latmap_metric_miou(ctx.h, _ptr(emb.contiguous()), _iptr(lab), emb.shape[0], emb.shape[1],
                                          _ptr(prototypes.contiguous()), c, inter.ctypes.data_as(C.c_void_p),
                                          uni.ctypes.data_as(C.c_void_p), C.byref(v)))
    return v.value, inter, uni


def metric_psnr(ctx, rendered, observed):
    """metric_psnr (io/metrics.hpp:28-33) -> (dB, exact)."""
    if rendered.numel() != observed.numel():
        raise _capi.InvalidArgument("metric_psnr: shape mismatch")
    db, ex = C.c_double(0), C.c_int32(0)
    check(ctx.h, lib().latmap_metric_psnr(ctx.h, _ptr(rendered.contiguous()), _ptr(observed.contiguous()),
                                          rendered.numel(), C.byref(db), C.byref(ex)))
    return db.value, bool(ex.value)


def query_map(ctx, features, atoms, proj, temperature, embedding):
    """query_map (io/evaluate.hpp:37-40): per-Gaussian cosine with one embedding (device)."""
    n, ds = features.shape
    k, df = atoms.shape
    out = torch.empty(n, device=features.device)
    check(ctx.h, lib().latmap_query_map(ctx.h, _ptr(features.contiguous()), n, ds, _ptr(atoms.contiguous()),
                                        _ptr(proj.contiguous()), k, df, float(temperature),
                                        _ptr(embedding.contiguous()), _ptr(out)))
    return out


def evaluate_map(ctx, m: GaussianMap, atoms, proj, temperature, frames, intr, prototypes=None, stride=1):
    """evaluate_map (evaluate.cpp:10-72) over device frames: each ``frames[f]`` has pose_rot,
    pose_trans, rgb (h x w x 3), assignment (h x w), features (n_set x df) and optionally labels
    (h x w, -1 = unlabeled), all torch CUDA tensors. Returns the reference's EvalResult fields."""
    if stride < 1:
        raise _capi.InvalidArgument("evaluate_map: stride must be >= 1")
    rows, cos_sum, psnr_sum = [], 0.0, 0.0
    c = 0 if prototypes is None else prototypes.shape[0]
    inter_all = np.zeros(c, np.int64)
    uni_all = np.zeros(c, np.int64)
    for fi in range(0, len(frames), stride):
        fr = frames[fi]
        out = render(ctx, m, make_pose(fr.pose_rot, fr.pose_trans), intr)
        row = {"frame_index": fi, "psnr": metric_psnr(ctx, out.color, fr.rgb)[0], "cos_loss": 0.0, "miou": 0.0,
               "labeled_pixels": 0}
        psnr_sum += row["psnr"]
        q, t, pix = gather_supervision(ctx, out.query, fr.assignment, fr.features, normalize=True)
        if q.shape[0] > 0:
            rec = reconstruct(ctx, q, atoms, proj, temperature)
            row["cos_loss"] = metric_cos(ctx, rec, t)[0]
            row["labeled_pixels"] = int(q.shape[0])
            labels = getattr(fr, "labels", None)
            if labels is not None and c > 0:
                miou, inter, uni = metric_miou(ctx, rec, labels.reshape(-1)[pix], prototypes)
                row["miou"] = miou
                inter_all += inter
                uni_all += uni
        cos_sum += row["cos_loss"]
        rows.append(row)
    nfr = len(rows)
    inc = uni_all > 0
    return {"cos_loss": cos_sum / nfr if nfr else 0.0, "psnr": psnr_sum / nfr if nfr else 0.0,
            "miou": float(np.mean(inter_all[inc] / uni_all[inc])) if inc.any() else 0.0, "frames": rows}


@dataclass
class AdamState:
    m: torch.Tensor
    v: torch.Tensor
    step: int = 0
    skipped: int = 0


def adam_step(ctx, param, grad, st: AdamState, lr):
    """adam_step (obj/adam.hpp:61-79); returns False when the block was skipped."""
    s, k, ap = C.c_int64(st.step), C.c_int64(st.skipped), C.c_int32(0)
    check(ctx.h, lib().latmap_adam_step(ctx.h, _ptr(param), _ptr(grad), _ptr(st.m), _ptr(st.v), param.numel(),
                                        C.byref(s), C.byref(k), float(lr), C.byref(ap)))
    st.step, st.skipped = s.value, k.value
    return bool(ap.value)


LOSS_TAIL = 16  # partials tail after the 8-double frame slots: trust, overflow, 8 Adam skip flags


def assemble_loss(partials, width, height, cfg) -> dict:
    """Host-side LossBreakdown of a batch from its loss-partials vector (latmap_loss_assemble;
    nframes = (len - 16) / 8 global frame slots followed by the 16-double tail). No device needed."""
    p = np.ascontiguousarray(partials, np.float64)
    nframes = (p.size - LOSS_TAIL) // 8
    out = LossBreakdown()
    check(None, lib().latmap_loss_assemble(p.ctypes.data_as(C.c_void_p), nframes, int(width), int(height),
                                            C.byref(cfg), C.byref(out)))
    return out.as_dict()


def default_config(**overrides) -> Config:
    c = Config()
    lib().latmap_default_config(C.byref(c))
    for kk, vv in overrides.items():
        setattr(c, kk, vv)
    return c


class Session:
    """Device-resident map + dictionary + Adam moments; one ``step`` = one Stage-I iteration."""

    def __init__(self, ctx: Context, cfg: Config, n, query_dim, k, embed_dim, intr):
        self.ctx, self.cfg, self.intr = ctx, cfg, intr
        self.ds, self.k, self.df = query_dim, k, embed_dim
        h = C.c_void_p()
        check(ctx.h, lib().latmap_session_create(ctx.h, C.byref(cfg), n, query_dim, k, embed_dim, C.byref(intr),
                                                 C.byref(h)))
        self.h = h
        self._keep = []
        self._owner = None

    @classmethod
    def _borrowed(cls, owner, ctx, cfg, h, query_dim, k, embed_dim, intr):
        """A view of a session owned by ``owner`` (a Pipeline): never destroyed here. The owner is
        held weakly (no reference cycle, so the owner is finalised while its context lives) and
        clears ``h`` when it goes."""
        s = cls.__new__(cls)
        s.ctx, s.cfg, s.intr, s.ds, s.k, s.df = ctx, cfg, intr, query_dim, k, embed_dim
        s.h, s._keep, s._owner = C.c_void_p(h), [], weakref.ref(owner)
        return s

    @property
    def n(self):
        return int(lib().latmap_session_size(self.h))

    def __del__(self):
        if getattr(self, "h", None) and getattr(self, "_owner", None) is None:
            try:
                lib().latmap_session_destroy(self.h)
            except TypeError:  # interpreter shutdown: the library handle is already gone
                pass
        self.h = None

    @staticmethod
    def _np_ptr(a):
        return a.ctypes.data_as(C.c_void_p) if a is not None else None

    def set_map(self, m):
        arrs = [np.ascontiguousarray(getattr(m, f), np.float32) for f in MAP_FIELDS]
        check(self.ctx.h, lib().latmap_session_set_map(self.h, *[self._np_ptr(a) for a in arrs]))
        self.ctx.sync()

    def get_map(self):
        out = [np.zeros((self.n, c), np.float32) for c in (3, 4, 3, 3)] + [np.zeros(self.n, np.float32),
                                                                            np.zeros((self.n, self.ds), np.float32)]
        check(self.ctx.h, lib().latmap_session_get_map(self.h, *[self._np_ptr(a) for a in out]))
        return dict(zip(MAP_FIELDS, out))

    def set_dictionary(self, atoms=None, anchor=None, proj=None):
        arrs = [None if a is None else np.ascontiguousarray(a, np.float32) for a in (atoms, anchor, proj)]
        check(self.ctx.h, lib().latmap_session_set_dictionary(self.h, *[self._np_ptr(a) for a in arrs]))
        self.ctx.sync()

    def stream_kmeans(self, batch, uniform, decay=1.0):
        """Dictionary maintenance (pipeline.cpp:201-205): stream_kmeans_update of the atoms /
        anchor / atom weights with the keyframe embeddings (host n x embed_dim), then the atoms'
        Adam moments reset. ``uniform`` as in Context.weighted_kmeans."""
        b = np.ascontiguousarray(batch, np.float32)
        if b.shape[0] and b.shape[1] != self.df:
            raise _capi.InvalidArgument("stream_kmeans_update: embedding dimension mismatch")
        fn, user, keep = _uniform_arg(uniform)
        check(self.ctx.h, lib().latmap_session_stream_kmeans(self.h, b.ctypes.data_as(C.c_void_p), b.shape[0],
                                                             float(decay), fn, user))
        del keep

    def dict_weights(self):
        out = np.zeros(self.k, np.float32)
        check(self.ctx.h, lib().latmap_session_get_dict_weights(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def set_dict_weights(self, w):
        w = np.ascontiguousarray(w, np.float32)
        check(self.ctx.h, lib().latmap_session_set_dict_weights(self.h, w.ctypes.data_as(C.c_void_p)))

    def get_anchor(self):
        out = np.zeros((self.k, self.df), np.float32)
        check(self.ctx.h, lib().latmap_session_get_anchor(self.h, self._np_ptr(out)))
        return out

    def get_dictionary(self):
        atoms = np.zeros((self.k, self.df), np.float32)
        proj = np.zeros((self.ds, self.df), np.float32)
        check(self.ctx.h, lib().latmap_session_get_dictionary(self.h, self._np_ptr(atoms), self._np_ptr(proj)))
        return atoms, proj

    def set_frames(self, frames):
        """frames: objects with pose_rot, pose_trans, rgb, depth, assignment, features (numpy, host).

        The arrays are copied H2D on the session stream; pinned (page-locked) numpy buffers keep
        the copies asynchronous."""
        cf = (Frame * len(frames))()
        keep = []
        for i, f in enumerate(frames):
            rgb = f.rgb if f.rgb.dtype == np.float32 and f.rgb.flags.c_contiguous else np.ascontiguousarray(f.rgb, np.float32)
            dep = f.depth if f.depth.dtype == np.float32 and f.depth.flags.c_contiguous else np.ascontiguousarray(f.depth, np.float32)
            asg = f.assignment if f.assignment.dtype == np.int32 and f.assignment.flags.c_contiguous else np.ascontiguousarray(f.assignment, np.int32)
            fea = f.features if f.features.dtype == np.float32 and f.features.flags.c_contiguous else np.ascontiguousarray(f.features, np.float32)
            keep.append((rgb, dep, asg, fea))
            cf[i] = Frame(make_pose(f.pose_rot, f.pose_trans), self._np_ptr(rgb), self._np_ptr(dep),
                          self._np_ptr(asg), self._np_ptr(fea), fea.shape[0])
        self._keep = keep
        check(self.ctx.h, lib().latmap_session_set_frames(self.h, len(frames), cf))

    def set_batch(self, global_batch, add_trust=True, slot_offset=0):
        check(self.ctx.h, lib().latmap_session_set_batch(self.h, int(global_batch), int(bool(add_trust))))
        check(self.ctx.h, lib().latmap_session_set_slot_offset(self.h, int(slot_offset)))

    def objective(self, want_grad=True, read=True):
        out = LossBreakdown()
        check(self.ctx.h, lib().latmap_session_objective(self.h, int(want_grad), C.byref(out) if read else None))
        return out.as_dict() if read else None

    def apply(self):
        check(self.ctx.h, lib().latmap_session_apply(self.h))

    def step(self, read=True):
        out = LossBreakdown()
        check(self.ctx.h, lib().latmap_session_step(self.h, C.byref(out) if read else None))
        return out.as_dict() if read else None

    def objective_ex(self, want_grad=True, map_grads=True, use_cached_renders=False, read=True):
        """total_objective with ObjectiveOptions (objective.hpp:33-43)."""
        out = LossBreakdown()
        check(self.ctx.h, lib().latmap_session_objective_ex(self.h, int(want_grad), int(map_grads),
                                                            int(use_cached_renders), C.byref(out) if read else None))
        return out.as_dict() if read else None

    def set_graphs(self, enable=True):
        """Replay captured CUDA graphs of the Stage-I step (default on)."""
        check(self.ctx.h, lib().latmap_session_set_graphs(self.h, int(bool(enable))))

    def step_dict(self, read=True):
        """One Stage-II iteration (pipeline.cpp:250-259): cached renders, dictionary-only Adam."""
        out = LossBreakdown()
        check(self.ctx.h, lib().latmap_session_step_dict(self.h, C.byref(out) if read else None))
        return out.as_dict() if read else None

    ROW = 14  # + query_dim: position 3 | rotation 4 | color 3 | log_scale 3 | opacity 1 | features

    def export_rows(self, out=None):
        """The map as device AoS rows (the store's record layout), a torch tensor [n, 14 + ds]."""
        if out is None:
            out = torch.empty((self.n, self.ROW + self.ds), dtype=torch.float32, device=f"cuda:{self.ctx.device}")
        check(self.ctx.h, lib().latmap_session_export_rows(self.h, C.c_void_p(out.data_ptr())))
        return out

    def import_rows(self, rows, kept=None):
        """Replace the map with device AoS ``rows``; Adam moments of old rows with kept[i] carry over
        to the first sum(kept) rows (MapOptimizer::keep_map_rows), the rest start at zero."""
        n_new = int(rows.shape[0])
        km = None if kept is None else np.ascontiguousarray(kept, np.uint8)
        n_kept = int(km.sum()) if km is not None else self.n
        check(self.ctx.h, lib().latmap_session_import_rows(self.h, C.c_void_p(rows.data_ptr()) if n_new else None,
                                                           n_new, self._np_ptr(km), n_kept))

    def import_rows_device(self, rows, kept, n_kept):
        """import_rows with the kept mask on the device (torch uint8/bool, one entry per old row) and
        its count known: no host pass over the rows."""
        n_new = int(rows.shape[0])
        km = None if kept is None else kept.to(torch.uint8).contiguous()
        check(self.ctx.h, lib().latmap_session_import_rows_device(
            self.h, C.c_void_p(rows.data_ptr()) if n_new else None, n_new,
            C.c_void_p(km.data_ptr()) if km is not None and km.numel() else None, int(n_kept) if km is not None else 0))

    def seed_candidates(self, frame=0):
        """seed_gaussians (pipeline.cpp:39-73) rows for `frame` (features zero), device [n, 14 + ds]."""
        w, h = self.intr.width, self.intr.height
        cap = ((w + 1) // 2) * ((h + 1) // 2)
        rows = torch.empty((cap, self.ROW + self.ds), dtype=torch.float32, device=f"cuda:{self.ctx.device}")
        n = C.c_int64()
        check(self.ctx.h, lib().latmap_session_seed_candidates(self.h, int(frame), C.c_void_p(rows.data_ptr()), cap,
                                                               C.byref(n)))
        return rows[:n.value]

    def append_rows(self, rows, features=None):
        """ActiveSet::append_newborns: append device AoS rows (features from host when given)."""
        f = None if features is None else np.ascontiguousarray(features, np.float32)
        r = rows.contiguous()
        check(self.ctx.h, lib().latmap_session_append_rows(self.h, C.c_void_p(r.data_ptr()), int(r.shape[0]),
                                                           self._np_ptr(f)))

    def read_loss_async(self, buf):
        """Enqueue the D2H copy of the step's loss partials into ``buf`` (pinned float64 numpy) on
        the context stream; after the stream passes this point, ``assemble_loss(buf[:n], ...)``
        gives the LossBreakdown. Returns n."""
        cnt = C.c_int64(0)
        check(self.ctx.h, lib().latmap_session_read_loss_async(self.h, buf.ctypes.data_as(C.c_void_p), buf.size,
                                                               C.byref(cnt)))
        return cnt.value

    def read_loss(self):
        out = LossBreakdown()
        check(self.ctx.h, lib().latmap_session_read_loss(self.h, C.byref(out)))
        return out.as_dict()

    def grad_buffer(self):
        p, n = C.c_void_p(), C.c_int64()
        check(self.ctx.h, lib().latmap_session_grad_buffer(self.h, C.byref(p), C.byref(n)))
        return _device_view(p.value, n.value, torch.float32, self.ctx.device, owner=self)

    def loss_buffer(self):
        p, n = C.c_void_p(), C.c_int64()
        check(self.ctx.h, lib().latmap_session_loss_buffer(self.h, C.byref(p), C.byref(n)))
        return _device_view(p.value, n.value, torch.float64, self.ctx.device, owner=self)

    def frame_images(self, b):
        ps = [C.c_void_p() for _ in range(4)]
        check(self.ctx.h, lib().latmap_session_frame_images(self.h, b, *[C.byref(p) for p in ps]))
        h, w = self.intr.height, self.intr.width
        shapes = [(h, w, 3), (h, w), (h, w, self.ds), (h, w)]
        return [_device_view(p.value, int(np.prod(s)), torch.float32, self.ctx.device, owner=self).view(*s)
                for p, s in zip(ps, shapes)]

    GRAD_BLOCKS = ("positions", "rotations", "colors", "log_scales", "opacity_logits", "features", "proj", "atoms")

    def grad_blocks(self):
        """{block name: (offset, length)} of the flat parameter / gradient / moment buffers (blocks
        start 16-byte aligned, so offsets are not a plain running sum)."""
        off = np.zeros(8, np.int64)
        ln = np.zeros(8, np.int64)
        check(self.ctx.h, lib().latmap_session_grad_layout(self.h, off.ctypes.data_as(C.c_void_p),
                                                          ln.ctypes.data_as(C.c_void_p)))
        return {nm: (int(o), int(n)) for nm, o, n in zip(self.GRAD_BLOCKS, off, ln)}

    def grad_block_views(self, flat=None):
        """The flat gradient buffer (or `flat`, same layout) split into its 8 named blocks."""
        flat = self.grad_buffer() if flat is None else flat
        return {nm: flat[o:o + n] for nm, (o, n) in self.grad_blocks().items()}

    def check_overflow(self):
        """After objective -> all-reduce -> apply: True when some rank's tile lists overflowed (every
        rank's Adam skipped the step; this rank's buffers are grown). Synchronises."""
        any_ = C.c_int32()
        check(self.ctx.h, lib().latmap_session_check_overflow(self.h, C.byref(any_)))
        return bool(any_.value)

    def overflow_steps(self):
        """Sticky count of Adam steps skipped because a tile list overflowed."""
        n = C.c_int64()
        check(self.ctx.h, lib().latmap_session_overflow_steps(self.h, C.byref(n)))
        return int(n.value)

    def shard_range(self, nranks, rank):
        b, e = C.c_int64(), C.c_int64()
        check(self.ctx.h, lib().latmap_session_shard_range(self.h, int(nranks), int(rank), C.byref(b), C.byref(e)))
        return b.value, e.value

    def shard_check(self, begin, end):
        check(self.ctx.h, lib().latmap_session_shard_check(self.h, int(begin), int(end)))

    def apply_range(self, begin, end):
        """Adam on the flat range [begin, end) with the all-reduced skip flags (sharded step)."""
        check(self.ctx.h, lib().latmap_session_apply_range(self.h, int(begin), int(end)))

    def params_buffer(self):
        p, n = C.c_void_p(), C.c_int64()
        check(self.ctx.h, lib().latmap_session_params_buffer(self.h, C.byref(p), C.byref(n)))
        return _device_view(p.value, n.value, torch.float32, self.ctx.device, owner=self)

    def sharded_step(self, exchange, read=False, attempts=3, apply=True):
        """One keyframe-sharded Stage-I iteration: this rank's objective (global batch
        mean, set_batch), ``exchange(self)`` summing gradients and loss partials over ranks (e.g.
        Comm.session_allreduce), then the identical Adam on every rank. With ``read`` the step is
        checked for a tile-list overflow on any rank and repeated (all ranks take the same branch:
        the flag is part of the summed partials) and the LossBreakdown is returned."""
        for _ in range(attempts):
            self.objective(want_grad=True, read=False)
            exchange(self)
            if apply:
                self.apply()
            if not read:
                return None
            if not self.check_overflow():
                return self.read_loss()
        raise _capi.LatmapError("sharded_step: tile-list overflow persisted")

    DECODER_PATHS = {0: "none", 1: "fp32", 2: "tc_fused", 3: "tc_staged"}

    def set_parity_export(self, enable=True):
        """Make the bf16 tcgen05 decoders also store each row's (|F_hat|^2, F_hat.F)."""
        check(self.ctx.h, lib().latmap_session_set_parity_export(self.h, int(bool(enable))))

    def decoder_export(self, attention=True, row_nd=True):
        """The last decoded frame's decoder path name, its attention P (rows x K, device) and
        per-row (nu^2, dot) as the tcgen05 kernels computed them (None where not requested)."""
        path, rows = C.c_int32(), C.c_int64()
        check(self.ctx.h, lib().latmap_session_decoder_export(self.h, C.byref(path), C.byref(rows), None, None))
        dev = f"cuda:{self.ctx.device}"
        p = torch.empty((rows.value, self.k), dtype=torch.float32, device=dev) if attention else None
        nd = torch.empty((rows.value, 2), dtype=torch.float32, device=dev) if row_nd else None
        if attention or row_nd:
            check(self.ctx.h, lib().latmap_session_decoder_export(
                self.h, None, None, C.c_void_p(p.data_ptr()) if p is not None else None,
                C.c_void_p(nd.data_ptr()) if nd is not None else None))
        return self.DECODER_PATHS[path.value], p, nd

    PHASES = ("bin", "raster_fwd", "image_losses", "decoder", "raster_bwd", "project_bwd", "adam", "misc")

    def profile(self, enable=True):
        check(self.ctx.h, lib().latmap_session_profile(self.h, int(enable)))

    def phase_times(self):
        ms = np.zeros(8, np.float64)
        cnt = np.zeros(8, np.int64)
        check(self.ctx.h, lib().latmap_session_phase_times(self.h, ms.ctypes.data_as(C.c_void_p),
                                                           cnt.ctypes.data_as(C.c_void_p)))
        return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(self.PHASES)}

    def stats(self, nframes):
        vis = np.zeros(nframes, np.int64)
        pairs = np.zeros(nframes, np.int64)
        check(self.ctx.h, lib().latmap_session_stats(self.h, vis.ctypes.data_as(C.c_void_p),
                                                     pairs.ctypes.data_as(C.c_void_p)))
        return vis, pairs


class _CudaArrayView:
    """__cuda_array_interface__ over library-owned device memory. It keeps `owner` (the Session /
    Pipeline that owns the memory) alive for as long as torch holds the view. A view must still be
    fetched again after a row-set change (import_rows / append_rows swap the parameter set)."""

    def __init__(self, ptr, count, typestr, owner=None):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (ptr, False), "version": 3}


def _device_view(ptr, count, dtype, device, owner=None):
    typestr = "<f4" if dtype == torch.float32 else "<f8"
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArrayView(ptr, count, typestr, owner), device=f"cuda:{device}")


# ----------------------------------------------------------------------------- voxel-hash store
def voxel_of(p, voxel_size):
    """voxel_of (voxel_hash.cpp:9-16), host."""
    pa = np.ascontiguousarray(p, np.float32)
    k = np.zeros(3, np.int32)
    lib().latmap_voxel_of(pa.ctypes.data_as(C.c_void_p), float(voxel_size), k.ctypes.data_as(C.c_void_p))
    return tuple(int(v) for v in k)


def hash_voxel(key, capacity):
    """hash_voxel (voxel_hash.cpp:18-23), host."""
    k = np.ascontiguousarray(key, np.int32)
    return lib().latmap_hash_voxel(k.ctypes.data_as(C.c_void_p), int(capacity))


class Store:
    """VoxelHashStore with a pinned, device-mapped record pool (store/voxel_hash.hpp:25-73)."""

    def __init__(self, ctx, capacity, query_dim):
        self.ctx, self.ds, self.rs = ctx, query_dim, 14 + query_dim
        self.capacity = int(capacity)
        h = C.c_void_p()
        check(ctx.h, lib().latmap_store_create(ctx.h, int(capacity), int(query_dim), C.byref(h)))
        self.h = h

    @classmethod
    def _borrowed(cls, owner, ctx, h, capacity, query_dim):
        st = cls.__new__(cls)
        st.ctx, st.ds, st.rs, st.capacity, st.h = ctx, query_dim, 14 + query_dim, int(capacity), C.c_void_p(h)
        st._owner = weakref.ref(owner)
        return st

    def __del__(self):
        if getattr(self, "h", None) and getattr(self, "_owner", None) is None:
            try:
                lib().latmap_store_destroy(self.h)
            except TypeError:  # interpreter shutdown: the library handle is already gone
                pass
        self.h = None

    def _check(self, st):
        if st != _capi.OK:
            msg = (lib().latmap_store_last_error(self.h) or b"").decode()
            if st == _capi.EINVAL:
                raise _capi.InvalidArgument(msg)
            raise _capi.LatmapError(msg)

    def size(self):
        return lib().latmap_store_size(self.h)

    def stats(self):
        o = np.zeros(5, np.int64)
        lib().latmap_store_stats(self.h, o.ctypes.data_as(C.c_void_p))
        return dict(zip(("inserted", "updated", "rejected_duplicate", "rejected_overflow", "probe_steps"), o.tolist()))

    def insert(self, key, rec):
        k = np.ascontiguousarray(key, np.int32)
        r = np.ascontiguousarray(rec, np.float32)
        return lib().latmap_store_insert(self.h, k.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p))

    def update(self, key, rec):
        k = np.ascontiguousarray(key, np.int32)
        r = np.ascontiguousarray(rec, np.float32)
        return bool(lib().latmap_store_update(self.h, k.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p)))

    def find(self, key):
        k = np.ascontiguousarray(key, np.int32)
        return lib().latmap_store_find(self.h, k.ctypes.data_as(C.c_void_p))

    def records(self):
        n = self.size()
        out = np.zeros((n, self.rs), np.float32)
        keys = np.zeros((n, 3), np.int32)
        if n:
            self._check(lib().latmap_store_get_records(self.h, 0, n, out.ctypes.data_as(C.c_void_p),
                                                       keys.ctypes.data_as(C.c_void_p)))
        return out, keys

    def insert_global(self, recs, voxel_size):
        r = np.ascontiguousarray(recs, np.float32).reshape(-1, self.rs)
        ins = C.c_int64(0)
        self._check(lib().latmap_store_insert_global(self.h, r.ctypes.data_as(C.c_void_p), r.shape[0],
                                                     float(voxel_size), C.byref(ins)))
        return ins.value

    def insert_keyed(self, keys, recs):
        """VoxelHashStore::insert of each row under its given key, in row order (rebuilding a
        dump, artifacts.cpp:54-63); returns the number inserted."""
        k = np.ascontiguousarray(keys, np.int32).reshape(-1, 3)
        r = np.ascontiguousarray(recs, np.float32).reshape(-1, self.rs)
        if k.shape[0] != r.shape[0]:
            raise _capi.InvalidArgument("insert_keyed: keys and records differ in count")
        ins = C.c_int64(0)
        self._check(lib().latmap_store_insert_keyed(self.h, k.ctypes.data_as(C.c_void_p), r.ctypes.data_as(C.c_void_p),
                                                    r.shape[0], C.byref(ins)))
        return ins.value

    def fetch_local(self, center, radius, gather=False):
        c = np.ascontiguousarray(center, np.float32)
        cnt = C.c_int64(0)
        cap = self.size() + 1
        org = np.zeros(cap, np.int64)
        d = torch.empty((cap, self.rs), device=f"cuda:{self.ctx.device}") if gather else None
        self._check(lib().latmap_store_fetch_local(self.h, c.ctypes.data_as(C.c_void_p), float(radius),
                                                   org.ctypes.data_as(C.c_void_p), cap, C.byref(cnt),
                                                   C.c_void_p(d.data_ptr()) if gather else None))
        n = cnt.value
        return (org[:n].copy(), d[:n]) if gather else org[:n].copy()

    def sync(self, d_active, origin, dirty, center, radius, voxel_size):
        """d_active: torch CUDA (n, 14+ds) records; returns (d_out, out_origin, kept_mask, stats)."""
        n = 0 if d_active is None else d_active.shape[0]
        org = np.ascontiguousarray(origin, np.int64)
        dty = np.ascontiguousarray(dirty, np.uint8)
        c = np.ascontiguousarray(center, np.float32)
        cap = self.size() + n + 1
        # output buffers sized for the worst case (every stored record in radius) are kept across
        # calls: a fresh ~1 GB device buffer and a zero-filled origin array per frame cost tens of ms
        if getattr(self, "_dout", None) is None or self._dout.shape[0] < cap:
            self._dout = torch.empty((cap + cap // 8, self.rs), device=f"cuda:{self.ctx.device}")
            self._oo = np.empty(cap + cap // 8, np.int64)
        d_out, oo = self._dout, self._oo
        kept = np.zeros(max(n, 1), np.uint8)
        st = np.zeros(5, np.int64)
        cnt = C.c_int64(0)
        dptr = C.c_void_p(d_active.data_ptr()) if n else None
        self._check(lib().latmap_store_sync(self.h, dptr, org.ctypes.data_as(C.c_void_p), dty.ctypes.data_as(C.c_void_p),
                                            n, c.ctypes.data_as(C.c_void_p), float(radius), float(voxel_size),
                                            C.c_void_p(d_out.data_ptr()), oo.ctypes.data_as(C.c_void_p), cap,
                                            kept.ctypes.data_as(C.c_void_p), st.ctypes.data_as(C.c_void_p),
                                            C.byref(cnt)))
        w = cnt.value
        stats = dict(zip(("written_back", "newborn_inserted", "newborn_rejected", "pruned", "fetched"), st.tolist()))
        return d_out[:w].clone(), oo[:w].copy(), kept[:n].astype(bool), stats

    def radius_scan(self, center, radius):
        """The device radius scan of fetch_local only (no readback, nothing waits)."""
        c = np.ascontiguousarray(center, np.float32)
        self._check(lib().latmap_store_fetch_local_device(self.h, c.ctypes.data_as(C.c_void_p), float(radius), None, 0,
                                                          None, None))

    def fetch_local_device(self, center, radius, gather=False):
        """fetch_local with device outputs: (origin int64 CUDA, records or None)."""
        c = np.ascontiguousarray(center, np.float32)
        cnt = C.c_int64(0)
        self._check(lib().latmap_store_fetch_local_device(self.h, c.ctypes.data_as(C.c_void_p), float(radius), None, 0,
                                                          None, C.byref(cnt)))
        n = cnt.value
        dev = f"cuda:{self.ctx.device}"
        org = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        rec = torch.empty((max(n, 1), self.rs), device=dev) if gather else None
        self._check(lib().latmap_store_fetch_local_device(self.h, c.ctypes.data_as(C.c_void_p), float(radius),
                                                          C.c_void_p(org.data_ptr()), n,
                                                          C.c_void_p(rec.data_ptr()) if gather else None,
                                                          C.byref(cnt)))
        return (org[:n], rec[:n]) if gather else org[:n]

    def sync_device(self, d_active, d_origin, d_dirty, center, radius, voxel_size):
        """sync with the per-row arrays on the device (latmap_store_sync_device): d_origin torch
        int64 CUDA (n), d_dirty torch uint8 CUDA (n) or None (every row dirty). Returns device
        (d_out, out_origin, kept) views and the stats dict; the output buffers are reused by the
        next call."""
        n = 0 if d_active is None else d_active.shape[0]
        c = np.ascontiguousarray(center, np.float32)
        cap = self.size() + n + 1
        dev = f"cuda:{self.ctx.device}"
        if getattr(self, "_ddout", None) is None or self._ddout.shape[0] < cap:
            self._ddout = torch.empty((cap + cap // 8, self.rs), device=dev)
            self._ddorg = torch.empty(cap + cap // 8, dtype=torch.int64, device=dev)
        if getattr(self, "_dkept", None) is None or self._dkept.numel() < max(n, 1):
            self._dkept = torch.empty(max(n, 1) + max(n, 1) // 4, dtype=torch.uint8, device=dev)
        st = np.zeros(5, np.int64)
        cnt = C.c_int64(0)
        org = d_origin.contiguous() if n else None
        dty = d_dirty.to(torch.uint8).contiguous() if (n and d_dirty is not None) else None
        self._check(lib().latmap_store_sync_device(
            self.h, C.c_void_p(d_active.data_ptr()) if n else None, C.c_void_p(org.data_ptr()) if n else None,
            C.c_void_p(dty.data_ptr()) if dty is not None else None, n, c.ctypes.data_as(C.c_void_p), float(radius),
            float(voxel_size), C.c_void_p(self._ddout.data_ptr()), C.c_void_p(self._ddorg.data_ptr()), cap,
            C.c_void_p(self._dkept.data_ptr()), st.ctypes.data_as(C.c_void_p), C.byref(cnt)))
        w = cnt.value
        stats = dict(zip(("written_back", "newborn_inserted", "newborn_rejected", "pruned", "fetched"), st.tolist()))
        return self._ddout[:w], self._ddorg[:w], self._dkept[:n], stats


def default_pipeline_config(**overrides) -> _capi.PipelineConfig:
    pc = _capi.PipelineConfig()
    lib().latmap_default_pipeline_config(C.byref(pc))
    for kk, vv in overrides.items():
        if kk == "dict_init" and isinstance(vv, str):
            vv = {"kmeans": 0, "random": 1}[vv]
        setattr(pc, kk, vv)
    return pc


def select_keyframe(frame_index, stride):
    """pipeline.cpp:14-17."""
    r = lib().latmap_select_keyframe(int(frame_index), int(stride))
    if r < 0:
        raise _capi.InvalidArgument("select_keyframe: stride must be >= 1")
    return bool(r)


class Pipeline:
    """PipelineState + process_keyframe (pipe/pipeline.hpp:82-107, pipeline.cpp:106-312) over the
    device session and store; ``session`` / ``store`` are views of the pipeline's own."""

    def __init__(self, ctx: Context, cfg: Config, pcfg, intr):
        self.ctx, self.cfg, self.pcfg, self.intr = ctx, cfg, pcfg, intr
        h = C.c_void_p()
        check(ctx.h, lib().latmap_pipeline_create(ctx.h, C.byref(cfg), C.byref(pcfg), C.byref(intr), C.byref(h)))
        self.h = h
        self.session = Session._borrowed(self, ctx, cfg, lib().latmap_pipeline_session(h), pcfg.query_dim,
                                         pcfg.dict_size, pcfg.embed_dim, intr)
        self.store = Store._borrowed(self, ctx, lib().latmap_pipeline_store(h), pcfg.hash_capacity, pcfg.query_dim)

    def __del__(self):
        if getattr(self, "h", None):
            for v in ("session", "store"):
                if getattr(self, v, None) is not None:
                    getattr(self, v).h = None
            try:
                lib().latmap_pipeline_destroy(self.h)
            except TypeError:  # interpreter shutdown: the library handle is already gone
                pass
            self.h = None

    def _check(self, st):
        if st != _capi.OK:
            msg = (lib().latmap_pipeline_last_error(self.h) or b"").decode()
            cmsg = (lib().latmap_ctx_last_error(self.ctx.h) or b"").decode()
            msg = msg or cmsg
            if st == _capi.EINVAL:
                raise _capi.InvalidArgument(msg)
            raise _capi.LatmapError(f"latmap status {st}: {msg}")

    def process_keyframe(self, kf, frame_index=None):
        """kf: host keyframe (pose_rot (w,x,y,z), pose_trans, rgb H x W x 3, depth H x W,
        assignment H x W, features n_set x embed_dim). Returns the KeyframeLog as a dict."""
        fi = int(getattr(kf, "frame_index", 0) if frame_index is None else frame_index)
        rgb = np.ascontiguousarray(kf.rgb, np.float32)
        dep = np.ascontiguousarray(kf.depth, np.float32)
        asg = np.ascontiguousarray(kf.assignment, np.int32)
        fea = np.ascontiguousarray(kf.features, np.float32)
        npx = self.intr.width * self.intr.height
        if rgb.size != npx * 3 or dep.size != npx or asg.size != npx:
            raise _capi.InvalidArgument("process_keyframe: image size does not match the intrinsics")
        n_set = fea.shape[0] if fea.ndim == 2 and fea.size else 0
        if n_set and fea.shape[1] != self.pcfg.embed_dim:
            raise _capi.InvalidArgument("process_keyframe: embedding dimension mismatch")
        f = Frame(make_pose(kf.pose_rot, kf.pose_trans), rgb.ctypes.data_as(C.c_void_p), dep.ctypes.data_as(C.c_void_p),
                  asg.ctypes.data_as(C.c_void_p), fea.ctypes.data_as(C.c_void_p) if n_set else None, n_set)
        log = _capi.KeyframeLog()
        self._check(lib().latmap_pipeline_process_keyframe(self.h, C.byref(f), fi, C.byref(log)))
        return log.as_dict()

    def inject_fault(self, stage):
        """Test hook: the next process_keyframe fails at stage 1 (after seeding), 2 (after Stage
        I/II) or 3 (after the sync) and is rolled back (latmap_pipeline_inject_fault)."""
        self._check(lib().latmap_pipeline_inject_fault(self.h, int(stage)))

    def flush(self):
        """run_pipeline's final flush (pipeline.cpp:318-330); returns the SyncStats."""
        st = np.zeros(5, np.int64)
        self._check(lib().latmap_pipeline_flush(self.h, st.ctypes.data_as(C.c_void_p)))
        return dict(zip(_capi.SYNC_FIELDS, st.tolist()))

    def state(self):
        o = np.zeros(6, np.int64)
        self._check(lib().latmap_pipeline_state(self.h, o.ctypes.data_as(C.c_void_p)))
        return {"keyframes_processed": int(o[0]), "peak_active": int(o[1]), "history": int(o[2]),
                "reservoir_seen": int(o[3]), "failed": bool(o[4]),
                "traveled": float(np.array([o[5]], np.int64).astype(np.int32).view(np.float32)[0])}

    def active_set(self):
        n = self.session.n
        org = np.zeros(n, np.int64)
        dty = np.zeros(n, np.uint8)
        self._check(lib().latmap_pipeline_active_set(self.h, org.ctypes.data_as(C.c_void_p),
                                                     dty.ctypes.data_as(C.c_void_p)))
        return org, dty


class Comm:
    """NCCL communicator of the sharded step (latmap_comm_*): rank 0 makes the unique id, the
    caller distributes it (any channel), every rank joins with its rank."""

    def __init__(self, ctx: Context, nranks, rank, uid: bytes):
        if len(uid) != 128:
            raise _capi.InvalidArgument("comm: unique id must be 128 bytes")
        self.ctx, self.nranks, self.rank = ctx, int(nranks), int(rank)
        h = C.c_void_p()
        buf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(ctx.h, lib().latmap_comm_init(ctx.h, self.nranks, self.rank, buf, C.byref(h)))
        self.h = h

    @staticmethod
    def unique_id(ctx: Context) -> bytes:
        buf = (C.c_uint8 * 128)()
        check(ctx.h, lib().latmap_comm_unique_id(ctx.h, buf))
        return bytes(buf)

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().latmap_comm_destroy(self.h)
            except TypeError:  # interpreter shutdown: the library handle is already gone
                pass
            self.h = None

    def allreduce(self, t: torch.Tensor):
        """In-place sum over ranks of a contiguous fp32 / fp64 CUDA tensor (context stream)."""
        if t.dtype not in (torch.float32, torch.float64) or not t.is_contiguous():
            raise _capi.InvalidArgument("comm.allreduce: contiguous fp32 or fp64 tensor expected")
        check(self.ctx.h, lib().latmap_comm_allreduce(self.h, C.c_void_p(t.data_ptr()), t.numel(),
                                                      0 if t.dtype == torch.float32 else 1))

    def session_allreduce(self, s: Session):
        """The sharded iteration's exchange: gradients and loss partials summed over ranks."""
        check(self.ctx.h, lib().latmap_session_allreduce(s.h, self.h))

    def session_exchange_sharded(self, s: Session):
        """ZeRO-1 exchange + step: reduce-scatter, shard check, partials all-reduce, Adam on the
        shard, all-gather (replaces session_allreduce + Session.apply)."""
        check(self.ctx.h, lib().latmap_session_exchange_sharded(s.h, self.h))
