"""Seeded synthetic workloads for BASELINE.json configs 0-4.

No public dataset is involved: every config is generated here from a per-config
seed (0x4C41544D00 + cfg). Targets (RGB, depth) are rendered from a perturbed copy
of the map by a caller-supplied ``render_fn(map, pose_rot, pose_trans, intr) ->
(color HxWx3, depth HxW, alpha HxW)`` so the same generator serves the oracle tests
(oracle renderer) and the GPU bench (device renderer).

Choices for values the configs leave open (documented in DESIGN.md):
  keys: W ~ N(0,1) (d_s x d_f) so the implied keys D W^T have unit-variance entries,
        temperature = sqrt(d_s), anchor = D;
  loss: lambda_l2 = 0, lambda_i2 = 0 ("1 - cos on features + L1 on RGB and depth");
        lambda_trust = 0.1 for configs 1-4 (config 1 "trust-region ... lambda=0.1");
  perturbation: sigma_p = 0.01 m on positions, sigma_c = 0.05 on colours (clipped);
  observed depth = rendered depth where rendered alpha > 0.5, else 0;
  Voronoi ties -> lower seed index; camera walk (config 2): 0.1 m steps in a direction
  uniform on the sphere, yaw +-5 deg about camera y per step.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Frame:
    pose_rot: tuple
    pose_trans: tuple
    rgb: np.ndarray
    depth: np.ndarray
    assignment: np.ndarray
    features: np.ndarray


@dataclass
class Intr:
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int


@dataclass
class HostMap:
    positions: np.ndarray
    rotations: np.ndarray
    colors: np.ndarray
    log_scales: np.ndarray
    opacity_logits: np.ndarray
    features: np.ndarray

    @property
    def n(self):
        return self.positions.shape[0]

    def copy(self):
        return HostMap(*[getattr(self, f).copy() for f in ("positions", "rotations", "colors", "log_scales",
                                                            "opacity_logits", "features")])


@dataclass
class Workload:
    cfg_id: int
    intr: Intr
    map: HostMap
    atoms: np.ndarray
    anchor: np.ndarray
    proj: np.ndarray
    temperature: float
    frames: list
    lambdas: dict = field(default_factory=dict)
    iterations: int = 1
    name: str = ""


SPECS = {
    # id: (W, H, fx, cx, cy, N, box_lo, box_hi, d_s, K, d_f, seeds, mix, frames)
    0: (320, 240, 300.0, 160.0, 120.0, 20_000, (-2, -1.5, 1), (2, 1.5, 6), 16, 64, 512, 16, 3, 1),
    1: (640, 480, 525.0, 320.0, 240.0, 200_000, (-4, -3, 0.5), (4, 3, 8), 32, 128, 768, 48, 3, 1),
    2: (640, 480, 525.0, 320.0, 240.0, 500_000, (-4, -3, 0.5), (4, 3, 8), 32, 256, 512, 48, 3, 8),
    4: (1280, 960, 1050.0, 640.0, 480.0, 300_000, (-4, -3, 0.5), (4, 3, 8), 64, 1024, 1024, 128, 5, 1),
}
NAMES = {0: "cfg0-320x240-N20k-d16-K64-D512-fp32", 1: "cfg1-640x480-N200k-d32-K128-D768",
         2: "cfg2-8x640x480-N500k-d32-K256-D512", 4: "cfg4-1280x960-N300k-d64-K1024-D1024"}


def seed_for(cfg_id):
    return 0x4C41544D00 + cfg_id


def random_map(rng, n, lo, hi, ds, dtype=np.float32):
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    pos = lo + rng.random((n, 3)) * (hi - lo)
    q = rng.standard_normal((n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    lsc = rng.normal(-3.5, 0.5, (n, 3))
    opa = rng.standard_normal(n)
    col = rng.random((n, 3))
    feat = rng.standard_normal((n, ds))
    return HostMap(*[np.ascontiguousarray(a, dtype) for a in (pos, q, col, lsc, opa, feat)])


def voronoi_assignment(rng, w, h, n_seeds, device=None):
    seeds = rng.random((n_seeds, 2)) * np.array([w, h])
    if device is not None:  # same float64 distances and first-minimum ties, evaluated with torch
        import torch

        ys, xs = torch.meshgrid(torch.arange(h, dtype=torch.float64, device=device),
                                torch.arange(w, dtype=torch.float64, device=device), indexing="ij")
        sd = torch.as_tensor(seeds, device=device)
        d = (xs.reshape(-1, 1) - sd[None, :, 0]) ** 2 + (ys.reshape(-1, 1) - sd[None, :, 1]) ** 2
        return torch.argmin(d, dim=1).to(torch.int32).cpu().numpy()
    ys, xs = np.mgrid[0:h, 0:w]
    px = np.stack([xs.ravel(), ys.ravel()], 1).astype(np.float64)
    best = np.zeros(px.shape[0], np.int32)
    chunk = 1 << 16
    for s in range(0, px.shape[0], chunk):
        d = ((px[s:s + chunk, None, :] - seeds[None, :, :]) ** 2).sum(-1)
        best[s:s + chunk] = np.argmin(d, axis=1)  # ties -> lower index
    return best


def cell_embeddings(rng, atoms, n_cells, mix):
    k = atoms.shape[0]
    out = np.zeros((n_cells, atoms.shape[1]), np.float64)
    for c in range(n_cells):
        idx = rng.choice(k, size=mix, replace=False)
        z = rng.standard_normal(mix) / 0.1
        wts = np.exp(z - z.max())
        wts /= wts.sum()
        v = wts @ atoms[idx].astype(np.float64)
        out[c] = v / np.linalg.norm(v)
    return out.astype(np.float32)


def yaw_quat(theta):
    return (math.cos(theta / 2), 0.0, math.sin(theta / 2), 0.0)


def camera_walk(rng, nframes, step=0.1, yaw_deg=5.0):
    poses = []
    t = np.zeros(3)
    th = 0.0
    for f in range(nframes):
        if f > 0:
            d = rng.standard_normal(3)
            t = t + step * d / np.linalg.norm(d)
            th += math.radians(rng.uniform(-yaw_deg, yaw_deg))
        poses.append((yaw_quat(th), tuple(float(v) for v in t)))
    return poses


def make_workload(cfg_id, render_fn, scale=1.0):
    """Build config `cfg_id`. ``scale`` < 1 shrinks N and the image (tests only)."""
    W, H, fx, cx, cy, N, lo, hi, ds, K, df, n_seeds, mix, nfr = SPECS[cfg_id]
    if scale != 1.0:
        W, H = max(16, int(W * scale)), max(16, int(H * scale))
        fx, cx, cy = fx * scale, W / 2, H / 2
        N = max(64, int(N * scale * scale))
    rng = np.random.default_rng(seed_for(cfg_id))
    intr = Intr(fx, fx, cx, cy, W, H)
    m = random_map(rng, N, lo, hi, ds)
    atoms = rng.standard_normal((K, df))
    atoms /= np.linalg.norm(atoms, axis=1, keepdims=True)
    atoms = atoms.astype(np.float32)
    proj = rng.standard_normal((ds, df)).astype(np.float32)
    temperature = float(np.float32(math.sqrt(ds)))
    poses = camera_walk(rng, nfr) if nfr > 1 else [((1.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0))]
    # perturbed copy for the RGB / depth targets
    pert = m.copy()
    pert.positions = (pert.positions + rng.normal(0, 0.01, pert.positions.shape)).astype(np.float32)
    pert.colors = np.clip(pert.colors + rng.normal(0, 0.05, pert.colors.shape), 0, 1).astype(np.float32)
    frames = []
    for (q, t) in poses:
        color, depth, alpha = render_fn(pert, q, t, intr)
        depth_obs = np.where(alpha > 0.5, depth, 0.0).astype(np.float32)
        assign = voronoi_assignment(rng, W, H, n_seeds)
        feats = cell_embeddings(rng, atoms, n_seeds, mix)
        frames.append(Frame(q, t, np.ascontiguousarray(color, np.float32), np.ascontiguousarray(depth_obs),
                            assign.reshape(H, W), feats))
    lambdas = dict(lambda_l2=0.0, lambda_i2=0.0, lambda_trust=0.2 if cfg_id == 0 else 0.1, softmax_temp=temperature)
    iters = {0: 1, 1: 100, 2: 1, 4: 20}[cfg_id]
    return Workload(cfg_id, intr, m, atoms, atoms.copy(), proj, temperature, frames, lambdas, iters,
                    NAMES[cfg_id] + ("" if scale == 1.0 else f"-scale{scale}"))


# ----------------------------------------------------------------------------- config 3
@dataclass
class Streaming:
    """Config 3 (BASELINE.json configs[3]): a host-resident global map
    of voxel-hashed records streamed through the GPU active set along a camera trajectory."""
    intr: Intr
    records: np.ndarray      # n_global x (14 + d_s) AoS, the store's record layout
    atoms: np.ndarray
    proj: np.ndarray
    temperature: float
    poses: list              # (quat, trans) per frame
    assignments: list        # per frame H x W int32 (Voronoi cells)
    features: list           # per frame n_seeds x d_f
    voxel_size: float = 0.01
    radius: float = 6.0
    capacity: int = 1 << 24
    iters_per_frame: int = 10
    lambdas: dict = field(default_factory=dict)
    name: str = ""


def look_quat(d):
    """Camera-to-world rotation (w, x, y, z) of a camera looking along the horizontal unit vector d
    with image-down = world -z (camera axes: x right, y down, z forward; synthetic.cpp:145)."""
    z = np.array([d[0], d[1], 0.0])
    z /= np.linalg.norm(z)
    y = np.array([0.0, 0.0, -1.0])
    x = np.cross(y, z)
    R = np.stack([x, y, z], 1)  # columns = camera axes in world coordinates
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    if tr > 0:
        s = math.sqrt(tr + 1.0) * 2
        q = (0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s)
    elif R[0, 0] > R[1, 1] and R[0, 0] > R[2, 2]:
        s = math.sqrt(1.0 + R[0, 0] - R[1, 1] - R[2, 2]) * 2
        q = ((R[2, 1] - R[1, 2]) / s, 0.25 * s, (R[0, 1] + R[1, 0]) / s, (R[0, 2] + R[2, 0]) / s)
    elif R[1, 1] > R[2, 2]:
        s = math.sqrt(1.0 + R[1, 1] - R[0, 0] - R[2, 2]) * 2
        q = ((R[0, 2] - R[2, 0]) / s, (R[0, 1] + R[1, 0]) / s, 0.25 * s, (R[1, 2] + R[2, 1]) / s)
    else:
        s = math.sqrt(1.0 + R[2, 2] - R[0, 0] - R[1, 1]) * 2
        q = ((R[1, 0] - R[0, 1]) / s, (R[0, 2] + R[2, 0]) / s, (R[1, 2] + R[2, 1]) / s, 0.25 * s)
    return tuple(float(v) for v in q)


def spline_path(rng, nframes, step, lo, hi, margin=8.0, height=4.5):
    """Seeded Catmull-Rom spline through random control points inside the volume, sampled every
    `step` metres of arc length; returns positions and horizontal tangents."""
    lo, hi = np.asarray(lo, np.float64), np.asarray(hi, np.float64)
    cps = lo[:2] + margin + rng.random((8, 2)) * (hi[:2] - lo[:2] - 2 * margin)
    pts = []
    for i in range(1, len(cps) - 2):
        p0, p1, p2, p3 = cps[i - 1], cps[i], cps[i + 1], cps[i + 2]
        for t in np.linspace(0, 1, 400, endpoint=False):
            t2, t3 = t * t, t * t * t
            pts.append(0.5 * (2 * p1 + (-p0 + p2) * t + (2 * p0 - 5 * p1 + 4 * p2 - p3) * t2 +
                              (-p0 + 3 * p1 - 3 * p2 + p3) * t3))
    pts = np.asarray(pts)
    seg = np.linalg.norm(np.diff(pts, axis=0), axis=1)
    arc = np.concatenate([[0.0], np.cumsum(seg)])
    s = np.arange(nframes) * step
    out_p, out_d = [], []
    for si in s:
        j = min(np.searchsorted(arc, si), len(pts) - 2)
        d = pts[j + 1] - pts[j]
        out_p.append(np.array([pts[j][0], pts[j][1], height]))
        out_d.append(d / np.linalg.norm(d))
    return out_p, out_d


def make_streaming(n_global=5_000_000, nframes=100, scale=1.0, seeds=48, mix=3, device=None):
    """Config 3: 1200x680 (fx = fy = 600, principal point at the centre: SURVEY Appendix B.5),
    100 frames 0.05 m apart on a seeded spline through a 60 x 60 x 9 m volume, n_global records
    uniform in it, record voxel 0.01 m with a 2^24-slot table (Appendix B.6), active radius 6 m,
    d_s = 32, K = 256, D = 1024, 10 iterations per frame. ``scale`` < 1 shrinks the image and
    the record count (tests)."""
    W, H, fx = 1200, 680, 600.0
    if scale != 1.0:
        W, H, fx = max(32, int(W * scale)), max(32, int(H * scale)), fx * scale
        n_global = max(1000, int(n_global * scale * scale))
    ds, K, df = 32, 256, 1024
    rng = np.random.default_rng(seed_for(3))
    intr = Intr(fx, fx, W / 2, H / 2, W, H)
    lo, hi = (0.0, 0.0, 0.0), (60.0, 60.0, 9.0)
    m = random_map(rng, n_global, lo, hi, ds)
    recs = np.concatenate([m.positions, m.rotations, m.colors, m.log_scales, m.opacity_logits[:, None],
                           m.features], axis=1).astype(np.float32)
    del m
    atoms = rng.standard_normal((K, df))
    atoms /= np.linalg.norm(atoms, axis=1, keepdims=True)
    atoms = atoms.astype(np.float32)
    proj = rng.standard_normal((ds, df)).astype(np.float32)
    temperature = float(np.float32(math.sqrt(ds)))
    pos, dirs = spline_path(rng, nframes, 0.05, lo, hi)
    poses = [(look_quat(d), tuple(float(v) for v in p)) for p, d in zip(pos, dirs)]
    assigns, feats = [], []
    for _ in range(nframes):
        assigns.append(voronoi_assignment(rng, W, H, seeds, device).reshape(H, W))
        feats.append(cell_embeddings(rng, atoms, seeds, mix))
    lambdas = dict(lambda_l2=0.0, lambda_i2=0.0, lambda_trust=0.1, softmax_temp=temperature)
    return Streaming(intr, np.ascontiguousarray(recs), atoms, proj, temperature, poses, assigns, feats,
                     lambdas=lambdas, name=f"cfg3-{nframes}f-{W}x{H}-G{n_global}-d32-K256-D1024"
                     + ("" if scale == 1.0 else f"-scale{scale}"))
