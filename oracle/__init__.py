"""CPU oracle for the LatentAM hot path — TEST INFRASTRUCTURE ONLY.

ctypes front end over ``oracle/_build/liblatmap_oracle.so`` (a C restatement of
the reference, see ``latmap_oracle.h``). Only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module, and only as the checker / the timed CPU reference, never as product code.

Parity pin: the reference C++ cannot be compiled here (Eigen3 and doctest are
absent); this restatement is pinned against the reference's own known-answer
tests, brute-force oracles and finite-difference checks (tests/test_oracle_*.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liblatmap_oracle.so")
_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _declare(_lib)
    return _lib


class Intr(C.Structure):
    _fields_ = [("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("width", C.c_int32), ("height", C.c_int32)]


class VoxelKey(C.Structure):
    _fields_ = [("ix", C.c_int32), ("iy", C.c_int32), ("iz", C.c_int32)]


def _mk_types(ct):
    class Map(C.Structure):
        _fields_ = [("n", C.c_int64), ("ds", C.c_int32)] + [
            (nm, C.POINTER(ct)) for nm in ("pos", "rot", "col", "lsc", "opa", "feat")]

    class Pose(C.Structure):
        _fields_ = [("rot", ct * 4), ("trans", ct * 3)]

    class Splat(C.Structure):
        _fields_ = [("mean", ct * 2), ("cov_inv", ct * 4), ("depth", ct), ("alpha", ct),
                    ("source", C.c_int32), ("x0", C.c_int32), ("x1", C.c_int32),
                    ("y0", C.c_int32), ("y1", C.c_int32)]

    class Loss(C.Structure):
        _fields_ = [(nm, ct) for nm in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust",
                                         "total")] + [
            ("supervised_rows", C.c_int64), ("depth_empty", C.c_int32),
            ("zero_norm_flagged", C.c_int32)]

    class Frame(C.Structure):
        _fields_ = [("pose", Pose), ("rgb", C.POINTER(ct)), ("depth", C.POINTER(ct)),
                    ("assignment", C.POINTER(C.c_int32)), ("features", C.POINTER(ct)),
                    ("n_set", C.c_int64)]

    class Cfg(C.Structure):
        _fields_ = [("segment_mode", C.c_int32), ("dict_grads", C.c_int32),
                    ("map_grads", C.c_int32)] + [
            (nm, ct) for nm in CFG_REAL_FIELDS] + [("dict_learn", C.c_int32)]

    return Map, Pose, Splat, Loss, Frame, Cfg


CFG_REAL_FIELDS = ("lambda_cos", "lambda_l2", "lambda_trust", "trust_delta", "lambda_i1", "lambda_i2",
                   "lambda_rgb", "lambda_depth", "lambda_feat", "lr_proj", "lr_dict", "lr_position",
                   "lr_rotation", "lr_color", "lr_log_scale", "lr_opacity", "lr_feature",
                   "scene_extent")

_TYPES = {np.float32: _mk_types(C.c_float), np.float64: _mk_types(C.c_double)}
_SUF = {np.float32: "_f32", np.float64: "_f64"}
_CT = {np.float32: C.c_float, np.float64: C.c_double}


def _declare(L):
    for dt in (np.float32, np.float64):
        s = _SUF[dt]
        ct = _CT[dt]
        P = C.POINTER(ct)
        Map, Pose, Splat, Loss, Frame, Cfg = _TYPES[dt]
        f = getattr(L, "lm_render" + s)
        f.argtypes = [C.POINTER(Map), C.POINTER(Pose), C.POINTER(Intr), C.c_int, P, P, P, P,
                      C.POINTER(Splat), C.c_int64, C.POINTER(C.c_int64)]
        f = getattr(L, "lm_render_backward" + s)
        f.argtypes = [C.POINTER(Map), C.POINTER(Pose), C.POINTER(Intr), C.POINTER(Splat), C.c_int64,
                      P, P, P, C.c_int, C.POINTER(Map)]
        f = getattr(L, "lm_project_gaussian" + s)
        f.argtypes = [P, P, P, ct, C.POINTER(Pose), C.POINTER(Intr), P, P, P]
        f = getattr(L, "lm_quat_to_rot" + s)
        f.argtypes = [P, P]
        f = getattr(L, "lm_ssim" + s)
        f.argtypes = [P, P, C.c_int, C.c_int, C.c_int, P]
        f.restype = ct
        f = getattr(L, "lm_rgb_loss" + s)
        f.argtypes = [P, P, C.c_int, C.c_int, C.c_int, ct, ct, C.c_int, P, P, P, P]
        f = getattr(L, "lm_depth_loss" + s)
        f.argtypes = [P, P, P, C.c_int64, C.c_int, P, P, C.POINTER(C.c_int32)]
        f = getattr(L, "lm_trust_region_penalty" + s)
        f.argtypes = [P, P, C.c_int64, C.c_int64, ct, P]
        f.restype = ct
        f = getattr(L, "lm_feature_loss" + s)
        f.argtypes = [P, P, C.c_int64, C.c_int64, P, P, C.c_int64, ct, ct, ct, ct, C.c_int, P, P,
                      P, P, P, P, C.POINTER(C.c_int32)]
        f = getattr(L, "lm_dictionary_checksum" + s)
        f.argtypes = [P, C.c_int64, C.c_int64, P, C.c_int64]
        f.restype = C.c_double
        f = getattr(L, "lm_reconstruct" + s)
        f.argtypes = [P, C.c_int64, C.c_int64, P, C.c_int64, C.c_int64, P, ct, P, P]
        f = getattr(L, "lm_reconstruct_backward" + s)
        f.argtypes = [P, P, C.c_int64, C.c_int64, P, C.c_int64, C.c_int64, P, ct, P, P, P, P]
        f = getattr(L, "lm_gather_supervision" + s)
        f.argtypes = [P, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int32), P, C.c_int64, C.c_int64,
                      C.c_int, P, P, C.POINTER(C.c_int64)]
        f.restype = C.c_int64
        f = getattr(L, "lm_total_objective" + s)
        f.argtypes = [C.POINTER(Map), P, P, P, C.c_int64, C.c_int64, ct, C.POINTER(Frame), C.c_int,
                      C.POINTER(Intr), C.POINTER(Cfg), C.c_int, C.c_int, C.POINTER(Map), P, P,
                      C.POINTER(Loss)]
        f = getattr(L, "lm_adam_step" + s)
        f.argtypes = [P, P, P, P, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64), ct]
        f = getattr(L, "lm_renorm_quats" + s)
        f.argtypes = [P, C.c_int64]
        f.restype = None
    L.lm_voxel_of.argtypes = [C.POINTER(C.c_float), C.c_float]
    L.lm_voxel_of.restype = VoxelKey
    L.lm_hash_voxel.argtypes = [VoxelKey, C.c_int64]
    L.lm_hash_voxel.restype = C.c_int64
    L.lm_store_create.argtypes = [C.c_int64, C.c_int32]
    L.lm_store_create.restype = C.c_void_p
    L.lm_store_destroy.argtypes = [C.c_void_p]
    L.lm_store_insert.argtypes = [C.c_void_p, VoxelKey, C.POINTER(C.c_float)]
    L.lm_store_insert.restype = C.c_int64
    L.lm_store_update.argtypes = [C.c_void_p, VoxelKey, C.POINTER(C.c_float)]
    L.lm_store_update.restype = C.c_int32
    L.lm_store_find.argtypes = [C.c_void_p, VoxelKey]
    L.lm_store_find.restype = C.c_int64
    L.lm_store_size.argtypes = [C.c_void_p]
    L.lm_store_size.restype = C.c_int64
    L.lm_store_check_unique_keys.argtypes = [C.c_void_p]
    L.lm_store_get_record.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_float)]
    L.lm_store_set_record.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_float)]
    L.lm_store_record_key.argtypes = [C.c_void_p, C.c_int64]
    UNI = C.CFUNCTYPE(C.c_double, C.c_void_p)
    for dt in (np.float32, np.float64):
        sfx, ct = _SUF[dt], _CT[dt]
        P = C.POINTER(ct)
        f = getattr(L, "lm_weighted_kmeans" + sfx)
        f.argtypes = [P, P, C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, P, C.c_int64, C.c_int, P, P,
                      C.POINTER(C.c_int)]
        f = getattr(L, "lm_stream_kmeans_update" + sfx)
        f.argtypes = [P, C.c_int64, C.c_int64, P, P, P, C.c_int64, C.c_void_p, C.c_void_p, ct]
    L.lm_mt64_seed.argtypes = [C.c_void_p, C.c_uint64]
    L.lm_oracle_set_gemm_threads.argtypes = [C.c_int]
    L.lm_oracle_set_gemm_threads.restype = None
    L.lm_expf_bits.argtypes = [C.c_uint64, C.c_int64, C.c_void_p, C.c_int]
    L.lm_expf_bits.restype = None
    L.lm_mt64_next.argtypes = [C.c_void_p]
    L.lm_mt64_next.restype = C.c_uint64
    L.lm_mt64_uniform01.argtypes = [C.c_void_p]
    L.lm_mt64_uniform01.restype = C.c_double
    PF, PI = C.POINTER(C.c_float), C.POINTER(C.c_int32)
    L.lm_metric_cos.argtypes = [PF, PF, C.c_int64, C.c_int64, PI]
    L.lm_metric_cos.restype = C.c_double
    L.lm_metric_miou.argtypes = [PF, PI, C.c_int64, C.c_int64, PF, C.c_int64, C.POINTER(C.c_int64),
                                 C.POINTER(C.c_int64)]
    L.lm_metric_miou.restype = C.c_double
    L.lm_metric_psnr.argtypes = [PF, PF, C.c_int64, PI]
    L.lm_metric_psnr.restype = C.c_double
    L.lm_query_scores.argtypes = [PF, C.c_int64, C.c_int64, PF, PF]
    L.lm_store_record_key.restype = VoxelKey
    L.lm_store_stats.argtypes = [C.c_void_p, C.POINTER(C.c_int64)]
    L.lm_insert_global.argtypes = [C.c_void_p, C.POINTER(C.c_float), C.c_int64, C.c_float]
    L.lm_insert_global.restype = C.c_int64
    L.lm_fetch_local.argtypes = [C.c_void_p, C.POINTER(C.c_float), C.c_float, C.POINTER(C.c_int64),
                                 C.c_int64]
    L.lm_fetch_local.restype = C.c_int64
    L.lm_sync.argtypes = [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_int64),
                          C.POINTER(C.c_uint8), C.c_int64, C.POINTER(C.c_float), C.c_float,
                          C.c_float, C.POINTER(C.c_float), C.POINTER(C.c_int64), C.c_int64,
                          C.POINTER(C.c_uint8), C.POINTER(C.c_int64)]
    L.lm_sync.restype = C.c_int64


def _p(a, ct=None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"]
    if ct is None:
        ct = _CT[a.dtype.type]
    return a.ctypes.data_as(C.POINTER(ct))


# --------------------------------------------------------------------------- data types
@dataclass
class GaussianMap:
    """GaussianMapT SoA (types.hpp:93-199); rows are primitives."""
    positions: np.ndarray
    rotations: np.ndarray
    colors: np.ndarray
    log_scales: np.ndarray
    opacity_logits: np.ndarray
    features: np.ndarray

    @property
    def n(self):
        return self.positions.shape[0]

    @property
    def ds(self):
        return self.features.shape[1]

    @property
    def dtype(self):
        return self.positions.dtype.type

    def astype(self, dt):
        return GaussianMap(*[np.ascontiguousarray(getattr(self, f).astype(dt)) for f in FIELDS])

    def copy(self):
        return GaussianMap(*[getattr(self, f).copy() for f in FIELDS])

    @staticmethod
    def zeros_like(m):
        return GaussianMap(*[np.zeros_like(getattr(m, f)) for f in FIELDS])

    def _cmap(self):
        Map = _TYPES[self.dtype][0]
        return Map(self.n, self.ds, *[_p(getattr(self, f)) for f in FIELDS])


FIELDS = ("positions", "rotations", "colors", "log_scales", "opacity_logits", "features")


def make_pose(rot=(1, 0, 0, 0), trans=(0, 0, 0), dtype=np.float32):
    Pose = _TYPES[dtype][1]
    return Pose((_CT[dtype] * 4)(*rot), (_CT[dtype] * 3)(*trans))


def make_intr(fx, fy, cx, cy, width, height):
    return Intr(fx, fy, cx, cy, width, height)


def splat_dtype(dtype):
    return np.dtype([("mean", dtype, 2), ("cov_inv", dtype, 4), ("depth", dtype), ("alpha", dtype),
                     ("source", np.int32), ("x0", np.int32), ("x1", np.int32), ("y0", np.int32),
                     ("y1", np.int32)], align=True)


# --------------------------------------------------------------------------- renderer
def quat_to_rot(q, dtype=np.float32):
    q = np.ascontiguousarray(q, dtype)
    r = np.zeros(9, dtype)
    rc = getattr(lib(), "lm_quat_to_rot" + _SUF[dtype])(_p(q), _p(r))
    if rc != 0:
        raise ValueError("quat_to_rot: zero-norm or non-finite quaternion")
    return r.reshape(3, 3)


def project_gaussian(pos, rot, lsc, opa, pose_rot, pose_trans, intr, dtype=np.float64):
    L = lib()
    a = [np.ascontiguousarray(x, dtype) for x in (pos, rot, lsc)]
    mean = np.zeros(2, dtype)
    cov = np.zeros(4, dtype)
    depth = np.zeros(1, dtype)
    pose = make_pose(pose_rot, pose_trans, dtype)
    rc = getattr(L, "lm_project_gaussian" + _SUF[dtype])(_p(a[0]), _p(a[1]), _p(a[2]), opa,
                                                         C.byref(pose), C.byref(intr), _p(mean),
                                                         _p(cov), _p(depth))
    if rc != 1:
        return None
    return mean, cov.reshape(2, 2), float(depth[0])


def render(m: GaussianMap, pose_rot, pose_trans, intr, threads=1):
    dt = m.dtype
    L = lib()
    h, w = intr.height, intr.width
    color = np.zeros((h, w, 3), dt)
    depth = np.zeros((h, w), dt)
    query = np.zeros((h, w, m.ds), dt)
    alpha = np.zeros((h, w), dt)
    Splat = _TYPES[dt][2]
    cap = m.n + 1
    splats = np.zeros(cap, splat_dtype(dt))
    assert splats.dtype.itemsize == C.sizeof(Splat)
    ns = C.c_int64(0)
    cmap = m._cmap()
    pose = make_pose(pose_rot, pose_trans, dt)
    rc = getattr(L, "lm_render" + _SUF[dt])(
        C.byref(cmap), C.byref(pose), C.byref(intr), threads, _p(color), _p(depth), _p(query),
        _p(alpha), splats.ctypes.data_as(C.POINTER(Splat)), cap, C.byref(ns))
    if rc != 0:
        raise ValueError("render: invalid intrinsics")
    return dict(color=color, depth=depth, query=query, alpha=alpha, splats=splats[: ns.value].copy())


def render_backward(m: GaussianMap, pose_rot, pose_trans, intr, splats, d_color=None, d_depth=None,
                    d_query=None, threads=1):
    dt = m.dtype
    Splat = _TYPES[dt][2]
    g = GaussianMap.zeros_like(m)
    cg = g._cmap()
    cmap = m._cmap()
    pose = make_pose(pose_rot, pose_trans, dt)
    sp = np.ascontiguousarray(splats)
    getattr(lib(), "lm_render_backward" + _SUF[dt])(
        C.byref(cmap), C.byref(pose), C.byref(intr), sp.ctypes.data_as(C.POINTER(Splat)), len(sp),
        _p(d_color), _p(d_depth), _p(d_query), threads, C.byref(cg))
    return g


# --------------------------------------------------------------------------- losses
def ssim(a, b, want_grad=False):
    dt = a.dtype.type
    h, w = a.shape[:2]
    c = a.shape[2] if a.ndim == 3 else 1
    da = np.zeros_like(a) if want_grad else None
    v = getattr(lib(), "lm_ssim" + _SUF[dt])(_p(a), _p(b), h, w, c, _p(da))
    return (v, da) if want_grad else v


def rgb_loss(rendered, observed, lambda_i1, lambda_i2, want_grad=True):
    dt = rendered.dtype.type
    h, w, c = rendered.shape
    grad = np.zeros_like(rendered)
    out = [np.zeros(1, dt) for _ in range(3)]
    getattr(lib(), "lm_rgb_loss" + _SUF[dt])(_p(rendered), _p(observed), h, w, c, lambda_i1, lambda_i2,
                                             int(want_grad), _p(grad), *[_p(o) for o in out])
    return dict(l1=out[0][0], ssim_loss=out[1][0], value=out[2][0], grad=grad if want_grad else None)


def depth_loss(rendered, observed, alpha, want_grad=True):
    dt = rendered.dtype.type
    grad = np.zeros_like(rendered)
    v = np.zeros(1, dt)
    fl = C.c_int32(0)
    getattr(lib(), "lm_depth_loss" + _SUF[dt])(_p(rendered), _p(observed), _p(alpha), rendered.size,
                                               int(want_grad), _p(grad), _p(v), C.byref(fl))
    return dict(value=v[0], flagged=bool(fl.value), grad=grad if want_grad else None)


def trust_region_penalty(atoms, anchor, delta, want_grad=False):
    dt = atoms.dtype.type
    g = np.zeros_like(atoms) if want_grad else None
    v = getattr(lib(), "lm_trust_region_penalty" + _SUF[dt])(_p(atoms), _p(anchor), atoms.shape[0],
                                                             atoms.shape[1], delta, _p(g))
    return (v, g) if want_grad else v


def feature_loss(rec, tgt, atoms, anchor, delta, lambda_cos, lambda_l2, lambda_trust, want_grad=True):
    dt = rec.dtype.type
    n, df = rec.shape
    d_rec = np.zeros_like(rec)
    d_at = np.zeros_like(atoms)
    o = [np.zeros(1, dt) for _ in range(4)]
    zf = C.c_int32(0)
    getattr(lib(), "lm_feature_loss" + _SUF[dt])(
        _p(rec), _p(tgt), n, df, _p(atoms), _p(anchor), atoms.shape[0], delta, lambda_cos, lambda_l2,
        lambda_trust, int(want_grad), _p(d_rec), _p(d_at), *[_p(x) for x in o], C.byref(zf))
    return dict(cos_term=o[0][0], l2_term=o[1][0], trust_term=o[2][0], value=o[3][0],
                zero_norm_flagged=bool(zf.value), d_reconstructed=d_rec, d_atoms_trust=d_at)


# --------------------------------------------------------------------------- decoder
def dictionary_checksum(atoms, proj):
    dt = atoms.dtype.type
    return getattr(lib(), "lm_dictionary_checksum" + _SUF[dt])(_p(atoms), atoms.shape[0], atoms.shape[1],
                                                               _p(proj), proj.shape[0])


def reconstruct(q, atoms, proj, temperature, want_attention=False):
    dt = q.dtype.type
    n, ds = q.shape
    k, df = atoms.shape
    out = np.zeros((n, df), dt)
    att = np.zeros((n, k), dt)
    rc = getattr(lib(), "lm_reconstruct" + _SUF[dt])(_p(q), n, ds, _p(atoms), k, df, _p(proj),
                                                     temperature, _p(out), _p(att))
    if rc != 0:
        raise ValueError("reconstruct: temperature must be > 0")
    return (out, att) if want_attention else out


def reconstruct_backward(q, attention, atoms, proj, temperature, d_rec):
    dt = q.dtype.type
    n, ds = q.shape
    k, df = atoms.shape
    dq = np.zeros_like(q)
    dp = np.zeros_like(proj)
    da = np.zeros_like(atoms)
    getattr(lib(), "lm_reconstruct_backward" + _SUF[dt])(
        _p(q), _p(attention), n, ds, _p(atoms), k, df, _p(proj), temperature, _p(d_rec), _p(dq),
        _p(dp), _p(da))
    return dict(d_queries=dq, d_proj=dp, d_atoms=da)


# --------------------------------------------------------------------------- objective
@dataclass
class Config:
    """Hot-path subset of latmap::Config (config.hpp:10-71) with reference defaults."""
    lambda_cos: float = 0.5
    lambda_l2: float = 0.5
    lambda_trust: float = 0.2
    trust_delta: float = 0.1
    lambda_i1: float = 0.2
    lambda_i2: float = 0.8
    lambda_rgb: float = 1.0
    lambda_depth: float = 0.1
    lambda_feat: float = 5.0
    lr_proj: float = 0.01
    lr_dict: float = 0.01
    lr_position: float = 1e-4
    lr_rotation: float = 1e-3
    lr_color: float = 2.5e-3
    lr_log_scale: float = 5e-3
    lr_opacity: float = 5e-2
    lr_feature: float = 2.5e-3
    scene_extent: float = 1.0
    dict_learn: bool = True
    segment_mode: bool = False

    def _c(self, dt, map_grads=True, dict_grads=True):
        Cfg = _TYPES[dt][5]
        # Config fields are float in the reference; T(cfg.x) widens the float value.
        vals = [float(np.float32(getattr(self, f))) for f in CFG_REAL_FIELDS]
        return Cfg(int(self.segment_mode), int(dict_grads), int(map_grads), *vals, int(self.dict_learn))


@dataclass
class Frame:
    pose_rot: tuple
    pose_trans: tuple
    rgb: np.ndarray
    depth: np.ndarray
    assignment: np.ndarray
    features: np.ndarray


@dataclass
class Dictionary:
    atoms: np.ndarray
    anchor: np.ndarray
    proj: np.ndarray
    temperature: float = 1.0


def total_objective(m: GaussianMap, d: Dictionary, frames, intr, cfg: Config, want_grad=True,
                    threads=1, map_grads=True, dict_grads=True):
    dt = m.dtype
    Map, Pose, Splat, Loss, Frame_, Cfg = _TYPES[dt]
    keep = []
    cfr = (Frame_ * len(frames))()
    for i, f in enumerate(frames):
        arrs = [np.ascontiguousarray(f.rgb, dt), np.ascontiguousarray(f.depth, dt),
                np.ascontiguousarray(f.assignment, np.int32), np.ascontiguousarray(f.features, dt)]
        keep.append(arrs)
        cfr[i] = Frame_(make_pose(f.pose_rot, f.pose_trans, dt), _p(arrs[0]), _p(arrs[1]),
                        _p(arrs[2], C.c_int32), _p(arrs[3]), arrs[3].shape[0])
    g = GaussianMap.zeros_like(m)
    dp = np.zeros_like(d.proj)
    da = np.zeros_like(d.atoms)
    out = Loss()
    cmap = m._cmap()
    cg = g._cmap()
    ccfg = cfg._c(dt, map_grads, dict_grads)
    k, df = d.atoms.shape
    getattr(lib(), "lm_total_objective" + _SUF[dt])(
        C.byref(cmap), _p(d.atoms), _p(d.anchor), _p(d.proj), k, df, d.temperature, cfr, len(frames),
        C.byref(intr), C.byref(ccfg), threads, int(want_grad), C.byref(cg), _p(dp), _p(da),
        C.byref(out))
    loss = {f: getattr(out, f) for f, _ in Loss._fields_}
    return loss, (g, dp, da)


@dataclass
class AdamState:
    m: np.ndarray
    v: np.ndarray
    step: int = 0
    skipped: int = 0


def adam_step(param, grad, st: AdamState, lr):
    dt = param.dtype.type
    s = C.c_int64(st.step)
    k = C.c_int64(st.skipped)
    ok = getattr(lib(), "lm_adam_step" + _SUF[dt])(_p(param), _p(grad), _p(st.m), _p(st.v), param.size,
                                                   C.byref(s), C.byref(k), lr)
    st.step, st.skipped = s.value, k.value
    return bool(ok)


def renorm_quats(rot):
    getattr(lib(), "lm_renorm_quats" + _SUF[rot.dtype.type])(_p(rot), rot.shape[0])


@dataclass
class MapOptimizer:
    """MapOptimizer::step_map/step_dict (pipeline.cpp:75-95) over numpy blocks."""
    states: dict = field(default_factory=dict)

    def _st(self, name, a):
        if name not in self.states:
            self.states[name] = AdamState(np.zeros_like(a), np.zeros_like(a))
        return self.states[name]

    def step_map(self, m: GaussianMap, g: GaussianMap, cfg: Config):
        lr_pos = float(np.float32(cfg.lr_position) * np.float32(cfg.scene_extent))
        adam_step(m.positions, g.positions, self._st("positions", m.positions), lr_pos)
        adam_step(m.rotations, g.rotations, self._st("rotations", m.rotations), cfg.lr_rotation)
        renorm_quats(m.rotations)
        adam_step(m.colors, g.colors, self._st("colors", m.colors), cfg.lr_color)
        adam_step(m.log_scales, g.log_scales, self._st("log_scales", m.log_scales), cfg.lr_log_scale)
        adam_step(m.opacity_logits, g.opacity_logits, self._st("opacity_logits", m.opacity_logits),
                  cfg.lr_opacity)
        adam_step(m.features, g.features, self._st("features", m.features), cfg.lr_feature)

    def step_dict(self, d: Dictionary, d_proj, d_atoms, cfg: Config):
        adam_step(d.proj, d_proj, self._st("proj", d.proj), cfg.lr_proj)
        if cfg.dict_learn:
            adam_step(d.atoms, d_atoms, self._st("atoms", d.atoms), cfg.lr_dict)


# --------------------------------------------------------------------------- store
def voxel_of(p, voxel_size):
    a = np.ascontiguousarray(p, np.float32)
    k = lib().lm_voxel_of(_p(a), voxel_size)
    return (k.ix, k.iy, k.iz)


def hash_voxel(key, capacity):
    return lib().lm_hash_voxel(VoxelKey(*key), capacity)


class Store:
    """VoxelHashStore (voxel_hash.hpp:25-73); records are flat rows of 14 + d_s floats."""

    def __init__(self, capacity, query_dim):
        self.h = lib().lm_store_create(capacity, query_dim)
        if not self.h:
            raise ValueError("VoxelHashStore: capacity must be > 0")
        self.ds = query_dim
        self.rs = 14 + query_dim

    def __del__(self):
        if getattr(self, "h", None):
            lib().lm_store_destroy(self.h)
            self.h = None

    def insert(self, key, rec):
        r = np.ascontiguousarray(rec, np.float32)
        return lib().lm_store_insert(self.h, VoxelKey(*key), _p(r))

    def update(self, key, rec):
        r = np.ascontiguousarray(rec, np.float32)
        return bool(lib().lm_store_update(self.h, VoxelKey(*key), _p(r)))

    def find(self, key):
        return lib().lm_store_find(self.h, VoxelKey(*key))

    def size(self):
        return lib().lm_store_size(self.h)

    def check_unique_keys(self):
        return bool(lib().lm_store_check_unique_keys(self.h))

    def record(self, i):
        r = np.zeros(self.rs, np.float32)
        lib().lm_store_get_record(self.h, i, _p(r))
        return r

    def records(self):
        n = self.size()
        out = np.zeros((n, self.rs), np.float32)
        for i in range(n):
            lib().lm_store_get_record(self.h, i, _p(out[i]))
        return out

    def record_key(self, i):
        k = lib().lm_store_record_key(self.h, i)
        return (k.ix, k.iy, k.iz)

    def stats(self):
        o = np.zeros(5, np.int64)
        lib().lm_store_stats(self.h, _p(o, C.c_int64))
        return dict(zip(("inserted", "updated", "rejected_duplicate", "rejected_overflow", "probe_steps"),
                        o.tolist()))

    def insert_global(self, recs, voxel_size):
        r = np.ascontiguousarray(recs, np.float32)
        return lib().lm_insert_global(self.h, _p(r), r.shape[0], voxel_size)

    def fetch_local(self, center, radius):
        c = np.ascontiguousarray(center, np.float32)
        cap = self.size() + 1
        org = np.zeros(cap, np.int64)
        n = lib().lm_fetch_local(self.h, _p(c), radius, _p(org, C.c_int64), cap)
        if n == -1:
            raise ValueError("fetch_local: radius must be > 0")
        return org[:n].copy()

    def sync(self, active_recs, origin, dirty, center, radius, voxel_size):
        a = np.ascontiguousarray(active_recs, np.float32).reshape(-1, self.rs)
        n = a.shape[0]
        org = np.ascontiguousarray(origin, np.int64)
        dty = np.ascontiguousarray(dirty, np.uint8)
        c = np.ascontiguousarray(center, np.float32)
        cap = self.size() + n + 1
        out = np.zeros((cap, self.rs), np.float32)
        oo = np.zeros(cap, np.int64)
        kept = np.zeros(max(n, 1), np.uint8)
        st = np.zeros(5, np.int64)
        w = lib().lm_sync(self.h, _p(a), _p(org, C.c_int64), _p(dty, C.c_uint8), n, _p(c), radius,
                          voxel_size, _p(out), _p(oo, C.c_int64), cap, _p(kept, C.c_uint8),
                          _p(st, C.c_int64))
        stats = dict(zip(("written_back", "newborn_inserted", "newborn_rejected", "pruned", "fetched"),
                         st.tolist()))
        return out[:w].copy(), oo[:w].copy(), kept[:n].astype(bool), stats


def map_to_records(m: GaussianMap):
    return np.concatenate([m.positions, m.rotations, m.colors, m.log_scales, m.opacity_logits[:, None],
                           m.features], axis=1).astype(np.float32)


def records_to_map(r, ds):
    r = np.asarray(r, np.float32)
    return GaussianMap(np.ascontiguousarray(r[:, 0:3]), np.ascontiguousarray(r[:, 3:7]),
                       np.ascontiguousarray(r[:, 7:10]), np.ascontiguousarray(r[:, 10:13]),
                       np.ascontiguousarray(r[:, 13]), np.ascontiguousarray(r[:, 14:14 + ds]))


# --------------------------------------------------------------------------- streaming k-means
class MT64(C.Structure):
    """std::mt19937_64 state (lm_mt64); ``uniform01`` is the C function pointer drawing
    std::uniform_real_distribution<double>(0, 1) from it (what k-means++ consumes)."""
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_int32)]

    def __init__(self, seed=5489):
        super().__init__()
        lib().lm_mt64_seed(C.byref(self), seed)

    def next(self):
        return int(lib().lm_mt64_next(C.byref(self)))

    def uniform01(self):
        return float(lib().lm_mt64_uniform01(C.byref(self)))

    @staticmethod
    def uniform01_fn():
        """Address of lm_mt64_uniform01 (a C callback double(void*))."""
        return C.cast(lib().lm_mt64_uniform01, C.c_void_p).value


def weighted_kmeans(points, weights, k, rng: MT64, warm=None, max_iters=10):
    """weighted_kmeans (stream_kmeans.cpp:94-157) -> (centers k x dim, weights k, iterations)."""
    dt = points.dtype.type
    pts = np.ascontiguousarray(points)
    w = np.ascontiguousarray(weights, dtype=dt)
    n, dim = pts.shape
    cen = np.zeros((k, dim), dt)
    cw = np.zeros(k, dt)
    it = C.c_int(0)
    wm = None if warm is None else np.ascontiguousarray(warm, dtype=dt)
    rc = getattr(lib(), "lm_weighted_kmeans" + _SUF[dt])(
        _p(pts), _p(w), n, dim, k, MT64.uniform01_fn(), C.cast(C.byref(rng), C.c_void_p), _p(wm),
        0 if wm is None else wm.shape[0], max_iters, _p(cen), _p(cw), C.byref(it))
    if rc != 0:
        raise ValueError("weighted_kmeans: k must be >= 1")
    return cen, cw, it.value


def stream_kmeans_update(batch, atoms, anchor, weights, rng: MT64, decay=1.0):
    """stream_kmeans_update (stream_kmeans.cpp:159-196); updates atoms / anchor / weights in place."""
    dt = atoms.dtype.type
    b = np.ascontiguousarray(batch, dtype=dt)
    n = b.shape[0]
    if n and b.shape[1] != atoms.shape[1]:
        raise ValueError("stream_kmeans_update: embedding dimension mismatch")
    getattr(lib(), "lm_stream_kmeans_update" + _SUF[dt])(
        _p(b), n, atoms.shape[1], _p(atoms), _p(anchor), _p(weights), atoms.shape[0], MT64.uniform01_fn(),
        C.cast(C.byref(rng), C.c_void_p), _CT[dt](decay))


# --------------------------------------------------------------------------- evaluation metrics
def metric_cos(rec, tgt):
    """metric_cos (metrics.cpp:8-24) -> (value, flagged)."""
    r = np.ascontiguousarray(rec, np.float32)
    t = np.ascontiguousarray(tgt, np.float32)
    if r.shape != t.shape:
        raise ValueError("metric_cos: shape mismatch")
    fl = C.c_int32(0)
    v = lib().lm_metric_cos(_p(r), _p(t), r.shape[0], r.shape[1] if r.ndim > 1 else 0, C.byref(fl))
    return float(v), bool(fl.value)


def metric_miou(emb, labels, protos):
    """metric_miou (metrics.cpp:26-73) -> (miou, intersection, union)."""
    e = np.ascontiguousarray(emb, np.float32)
    lab = np.ascontiguousarray(labels, np.int32)
    p = np.ascontiguousarray(protos, np.float32)
    c = p.shape[0]
    inter = np.zeros(c, np.int64)
    uni = np.zeros(c, np.int64)
    v = lib().lm_metric_miou(_p(e), lab.ctypes.data_as(C.POINTER(C.c_int32)), e.shape[0], e.shape[1], _p(p), c,
                             inter.ctypes.data_as(C.POINTER(C.c_int64)), uni.ctypes.data_as(C.POINTER(C.c_int64)))
    if v < 0:
        raise ValueError("metric_miou: label id out of range")
    return float(v), inter, uni


def metric_psnr(a, b):
    """metric_psnr (metrics.cpp:75-89) -> (dB, exact)."""
    x = np.ascontiguousarray(a, np.float32).reshape(-1)
    y = np.ascontiguousarray(b, np.float32).reshape(-1)
    if x.shape != y.shape:
        raise ValueError("metric_psnr: shape mismatch")
    ex = C.c_int32(0)
    v = lib().lm_metric_psnr(_p(x), _p(y), x.shape[0], C.byref(ex))
    return float(v), bool(ex.value)


def query_scores(rec, embedding):
    """query_map (evaluate.cpp:74-88) scores of reconstructed rows against one embedding."""
    r = np.ascontiguousarray(rec, np.float32)
    e = np.ascontiguousarray(embedding, np.float32)
    out = np.zeros(r.shape[0], np.float32)
    lib().lm_query_scores(_p(r), r.shape[0], r.shape[1], _p(e), _p(out))
    return out


def set_gemm_threads(n):
    """Row-split threads for the oracle's dense products (results are bit-identical for any n)."""
    lib().lm_oracle_set_gemm_threads(int(n))


def expf_bits(first, n, threads=1):
    """libm expf (the reference's std::exp(float)) of the floats with bit patterns first + i."""
    out = np.empty(int(n), np.float32)
    lib().lm_expf_bits(int(first), int(n), out.ctypes.data_as(C.c_void_p), int(threads))
    return out
