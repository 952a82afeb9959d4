"""TEST INFRASTRUCTURE, NOT PRODUCT CODE: ctypes front end of the REFERENCE library itself.

oracle/ref/Makefile compiles /root/reference/proj/src unmodified against the from-scratch Eigen /
doctest stand-ins (oracle/stand_ins) into oracle/_ref/ (git-ignored; shipped to the GPU box with
the snapshot). oracle/ref/ref_capi.cpp exposes render<float>, total_objective<float> and a
Stage-I iteration (total_objective + MapOptimizer::step_map + step_dict, pipeline.cpp:236-246)
on raw arrays. Uses: pin the C restatement (oracle/latmap_oracle.c) bit for bit, and the
`reference` CPU baseline of bench.py. Only tests/, smoke() and bench.py's CPU legs import it.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "liblatmap_ref_capi.so")
_lib = None


class Map(C.Structure):
    _fields_ = [("n", C.c_int64), ("ds", C.c_int32)] + [(f, C.c_void_p) for f in (
        "positions", "rotations", "colors", "log_scales", "opacity_logits", "features")]


class Frame(C.Structure):
    _fields_ = [("pose", C.c_float * 7), ("rgb", C.c_void_p), ("depth", C.c_void_p), ("assignment", C.c_void_p),
                ("features", C.c_void_p), ("n_set", C.c_int64)]


class Intr(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


CFG_FIELDS = ("trust_delta", "lambda_cos", "lambda_l2", "lambda_trust", "lambda_i1", "lambda_i2", "lambda_rgb",
              "lambda_depth", "lambda_feat", "lr_proj", "lr_dict", "lr_position", "lr_rotation", "lr_color",
              "lr_log_scale", "lr_opacity", "lr_feature", "scene_extent", "softmax_temp")
# latmap::Config defaults (proj/include/latmap/core/config.hpp:18-40)
CFG_DEFAULTS = dict(trust_delta=0.1, lambda_cos=0.5, lambda_l2=0.5, lambda_trust=0.2, lambda_i1=0.2, lambda_i2=0.8,
                    lambda_rgb=1.0, lambda_depth=0.1, lambda_feat=5.0, lr_proj=0.01, lr_dict=0.01, lr_position=1e-4,
                    lr_rotation=1e-3, lr_color=2.5e-3, lr_log_scale=5e-3, lr_opacity=5e-2, lr_feature=2.5e-3,
                    scene_extent=1.0, softmax_temp=1.0)


class Config(C.Structure):
    _fields_ = [(f, C.c_float) for f in CFG_FIELDS] + [("dict_learn", C.c_int32), ("segment_mode", C.c_int32),
                                                        ("num_threads", C.c_int32)]


class PipelineConfig(C.Structure):
    """latmap_ref_pipeline_config: the pipeline fields of latmap::Config, api.PipelineConfig's order."""
    _fields_ = [("query_dim", C.c_int32), ("embed_dim", C.c_int32), ("dict_size", C.c_int32),
                ("stage1_iters", C.c_int32), ("stage2_iters", C.c_int32), ("history_sample", C.c_int32),
                ("history_capacity", C.c_int32), ("voxel_size", C.c_float), ("local_radius", C.c_float),
                ("sync_distance", C.c_float), ("hash_capacity", C.c_int64), ("local_mapping", C.c_int32),
                ("keyframe_stride", C.c_int32), ("seed", C.c_uint64), ("dict_init", C.c_int32),
                ("dict_decay", C.c_float), ("trust_anchor_persistent", C.c_int32)]


class Loss(C.Structure):
    _fields_ = [(f, C.c_float) for f in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust", "total")] + [
        ("supervised_rows", C.c_int64), ("depth_empty", C.c_int32), ("zero_norm_flagged", C.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class KeyframeLog(C.Structure):
    _fields_ = [("frame_index", C.c_int32), ("loss", Loss), ("seeded", C.c_int64), ("active_count", C.c_int64),
                ("global_count", C.c_int64), ("dict_weight_mass", C.c_double), ("synced", C.c_int32),
                ("sync", C.c_int64 * 5)]

    def as_dict(self):
        return {"frame_index": self.frame_index, "loss": self.loss.as_dict(), "seeded": self.seeded,
                "active_count": self.active_count, "global_count": self.global_count,
                "dict_weight_mass": self.dict_weight_mass, "synced": bool(self.synced),
                "sync": dict(zip(("written_back", "newborn_inserted", "newborn_rejected", "pruned", "fetched"),
                                 list(self.sync)))}


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle/ref; needs /root/reference)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.latmap_ref_last_error.restype = C.c_char_p
        L.latmap_ref_render.argtypes = [C.POINTER(Map), C.c_float * 7, C.POINTER(Intr), C.c_int32, P, P, P, P]
        L.latmap_ref_total_objective.argtypes = [C.POINTER(Map), P, P, P, C.c_int64, C.c_int32, C.c_float,
                                                 C.POINTER(Frame), C.c_int32, C.POINTER(Intr), C.POINTER(Config),
                                                 C.c_int32, C.POINTER(Loss), P, P, P]
        L.latmap_ref_session_create.argtypes = [C.POINTER(Map), P, P, P, C.c_int64, C.c_int32, C.c_float,
                                                C.POINTER(Frame), C.c_int32, C.POINTER(Intr), C.POINTER(Config),
                                                C.c_int32]
        L.latmap_ref_session_create.restype = P
        L.latmap_ref_session_step.argtypes = [P, C.POINTER(Loss)]
        L.latmap_ref_session_objective.argtypes = [P, C.POINTER(Loss)]
        L.latmap_ref_session_get.argtypes = [P, P, P, P]
        L.latmap_ref_session_destroy.argtypes = [P]
        L.latmap_ref_pipeline_create.argtypes = [C.POINTER(Config), C.POINTER(PipelineConfig), C.POINTER(Intr)]
        L.latmap_ref_pipeline_create.restype = P
        L.latmap_ref_pipeline_process.argtypes = [P, C.POINTER(Frame), C.c_int32, C.POINTER(KeyframeLog)]
        L.latmap_ref_pipeline_flush.argtypes = [P, P]
        L.latmap_ref_pipeline_get.argtypes = [P, P, P, P, P, P]
        L.latmap_ref_pipeline_get.restype = C.c_int64
        L.latmap_ref_pipeline_destroy.argtypes = [P]
        _lib = L
    return _lib


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _f32(a):
    return np.ascontiguousarray(a, np.float32)


class _Keep:
    """Holds the contiguous copies the C structs point into."""

    def __init__(self):
        self.arrs = []

    def __call__(self, a, dt=np.float32):
        a = np.ascontiguousarray(a, dt)
        self.arrs.append(a)
        return a


def _map(m, keep):
    arrs = [keep(getattr(m, f)) for f in ("positions", "rotations", "colors", "log_scales", "opacity_logits",
                                          "features")]
    n = arrs[0].shape[0]
    ds = arrs[5].shape[1] if arrs[5].ndim == 2 else 0
    return Map(n, ds, *[a.ctypes.data for a in arrs])


def _intr(i):
    return Intr(i.fx, i.fy, i.cx, i.cy, i.width, i.height)


def _pose(q, t):
    return (C.c_float * 7)(*[float(v) for v in q], *[float(v) for v in t])


def _frames(frames, keep):
    arr = (Frame * len(frames))()
    for i, f in enumerate(frames):
        feats = keep(f.features)
        arr[i] = Frame(_pose(f.pose_rot, f.pose_trans), keep(f.rgb).ctypes.data, keep(f.depth).ctypes.data,
                       keep(f.assignment, np.int32).ctypes.data, feats.ctypes.data, feats.shape[0])
    return arr


def make_config(num_threads=1, dict_learn=True, segment_mode=False, **over):
    vals = dict(CFG_DEFAULTS)
    vals.update({k: v for k, v in over.items() if k in CFG_DEFAULTS})
    return Config(*[float(np.float32(vals[f])) for f in CFG_FIELDS], int(dict_learn), int(segment_mode),
                  int(num_threads))


def _check(rc):
    if rc != 0:
        raise RuntimeError(lib().latmap_ref_last_error().decode())


def render(m, q, t, intr, threads=1):
    keep = _Keep()
    cm = _map(m, keep)
    h, w = intr.height, intr.width
    ds = cm.ds
    out = {"color": np.zeros((h, w, 3), np.float32), "depth": np.zeros((h, w), np.float32),
           "query": np.zeros((h, w, ds), np.float32), "alpha": np.zeros((h, w), np.float32)}
    ci = _intr(intr)
    _check(lib().latmap_ref_render(C.byref(cm), _pose(q, t), C.byref(ci), threads, _p(out["color"]),
                                   _p(out["depth"]), _p(out["query"]), _p(out["alpha"])))
    return out


def total_objective(m, atoms, anchor, proj, temperature, frames, intr, cfg: Config, threads=1, want_grad=True):
    keep = _Keep()
    cm = _map(m, keep)
    atoms, anchor, proj = keep(atoms), keep(anchor), keep(proj)
    k, df = atoms.shape
    fr = _frames(frames, keep)
    ci = _intr(intr)
    loss = Loss()
    n, ds = cm.n, cm.ds
    g = np.zeros(n * (14 + ds), np.float32) if want_grad else None
    dp = np.zeros((ds, df), np.float32) if want_grad else None
    da = np.zeros((k, df), np.float32) if want_grad else None
    _check(lib().latmap_ref_total_objective(C.byref(cm), _p(atoms), _p(anchor), _p(proj), k, df, float(temperature),
                                            fr, len(frames), C.byref(ci), C.byref(cfg), threads, C.byref(loss),
                                            _p(g), _p(dp), _p(da)))
    return loss.as_dict(), (g, dp, da)


class Session:
    """The reference's Stage-I iteration on persistent state (for timing and step parity)."""

    def __init__(self, m, atoms, anchor, proj, temperature, frames, intr, cfg: Config, threads=1):
        keep = _Keep()
        cm = _map(m, keep)
        atoms, anchor, proj = keep(atoms), keep(anchor), keep(proj)
        self.k, self.df = atoms.shape
        self.n, self.ds = cm.n, cm.ds
        fr = _frames(frames, keep)
        ci = _intr(intr)
        self.h = lib().latmap_ref_session_create(C.byref(cm), _p(atoms), _p(anchor), _p(proj), self.k, self.df,
                                                 float(temperature), fr, len(frames), C.byref(ci), C.byref(cfg),
                                                 threads)
        if not self.h:
            raise RuntimeError(lib().latmap_ref_last_error().decode())

    def step(self):
        loss = Loss()
        _check(lib().latmap_ref_session_step(self.h, C.byref(loss)))
        return loss.as_dict()

    def objective(self):
        """total_objective with gradients, no optimiser step."""
        loss = Loss()
        _check(lib().latmap_ref_session_objective(self.h, C.byref(loss)))
        return loss.as_dict()

    def get(self):
        m = np.zeros(self.n * (14 + self.ds), np.float32)
        a = np.zeros((self.k, self.df), np.float32)
        p = np.zeros((self.ds, self.df), np.float32)
        lib().latmap_ref_session_get(self.h, _p(m), _p(a), _p(p))
        return m, a, p

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().latmap_ref_session_destroy(self.h)
            except Exception:  # noqa: BLE001  interpreter shutdown
                pass
            self.h = None


class Pipeline:
    """The reference's keyframe pipeline (PipelineState / process_keyframe and run_pipeline's final
    flush, pipeline.cpp:106-330) on host arrays."""

    def __init__(self, cfg: Config, pc: PipelineConfig, intr):
        self.pc = pc
        self.intr = _intr(intr)
        self.h = lib().latmap_ref_pipeline_create(C.byref(cfg), C.byref(pc), C.byref(self.intr))
        if not self.h:
            raise RuntimeError(lib().latmap_ref_last_error().decode())

    def process_keyframe(self, kf):
        keep = _Keep()
        fr = _frames([kf], keep)
        log = KeyframeLog()
        _check(lib().latmap_ref_pipeline_process(self.h, fr, int(getattr(kf, "frame_index", 0)), C.byref(log)))
        return log.as_dict()

    def flush(self):
        st = np.zeros(5, np.int64)
        _check(lib().latmap_ref_pipeline_flush(self.h, _p(st)))
        return dict(zip(("written_back", "newborn_inserted", "newborn_rejected", "pruned", "fetched"), st.tolist()))

    def state(self):
        n = lib().latmap_ref_pipeline_get(self.h, None, None, None, None, None)
        org = np.zeros(max(n, 1), np.int64)
        k, ds, df = self.pc.dict_size, self.pc.query_dim, self.pc.embed_dim
        atoms = np.zeros((k, df), np.float32)
        proj = np.zeros((ds, df), np.float32)
        w = np.zeros(k, np.float32)
        size = C.c_int64(0)
        lib().latmap_ref_pipeline_get(self.h, _p(org), _p(atoms), _p(proj), _p(w), C.byref(size))
        return {"origin": org[:n], "atoms": atoms, "proj": proj, "weights": w, "store_size": size.value}

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().latmap_ref_pipeline_destroy(self.h)
            except Exception:  # noqa: BLE001
                pass
            self.h = None
