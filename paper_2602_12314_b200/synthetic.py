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


def voronoi_assignment(rng, w, h, n_seeds):
    seeds = rng.random((n_seeds, 2)) * np.array([w, h])
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
