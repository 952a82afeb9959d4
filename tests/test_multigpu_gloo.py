"""The N>1 keyframe-sharded path on CPU: 2 ranks over gloo.

1. The LIBRARY's host side of the exchange: every rank writes its frames' loss partials into the
   global slots rank_plan assigns (slot_offset), rank 0 alone the trust slot; the partial vectors
   are summed with all_reduce and the library's own assembly (latmap_loss_assemble, the code the
   device step runs) must give the full batch's LossBreakdown (objective.cpp:77,187-190).
2. The sharding identity itself: per-shard gradients with the global batch mean, trust term once,
   summed over ranks == the full-batch gradient of total_objective (objective.cpp:67-194). The
   device objective needs a GPU, so the CPU oracle evaluates each shard here; the library's
   sharded device path is tested on one GPU in tests/test_gpu_sharded.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2602_12314_b200.sharding import rank_plan, shard_frames
from tests.helpers import random_map, small_intrinsics


def test_shard_frames_partition():
    for nf in (1, 5, 8):
        for world in (1, 2, 3, 4, 8):
            if world > nf:
                continue
            got = []
            for r in range(world):
                f, c = shard_frames(nf, world, r)
                got += list(range(f, f + c))
            assert got == list(range(nf))
    p = rank_plan(8, 4, 2)
    assert p["frames"] == [4, 5] and p["global_batch"] == 8 and not p["add_trust"] and p["slot_offset"] == 4


def _problem():
    rng = np.random.default_rng(99)
    intr = small_intrinsics(12, 12, 14.0)
    m = random_map(10, 4, rng)
    atoms = rng.standard_normal((6, 12)) * 0.5
    d = oracle.Dictionary(atoms + 0.05, atoms.copy(), rng.standard_normal((4, 12)) * 0.5, 1.0)
    frames = []
    for k in range(4):
        feats = rng.standard_normal((144, 12))
        feats /= np.linalg.norm(feats, axis=1, keepdims=True)
        frames.append(oracle.Frame((1, 0, 0, 0), (0.03 * k, 0.0, 0.0), rng.random((12, 12, 3)),
                                   1 + 2 * rng.random((12, 12)), np.arange(144, dtype=np.int32), feats))
    return intr, m, d, frames


def _flat(g, dp, da):
    return np.concatenate([getattr(g, f).reshape(-1) for f in oracle.FIELDS] + [dp.reshape(-1), da.reshape(-1)])


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    intr, m, d, frames = _problem()
    plan = rank_plan(len(frames), world, rank)
    cfg = oracle.Config()
    mine = [frames[i] for i in plan["frames"]]
    _, (g, dp, da) = oracle.total_objective(m, d, mine, intr, cfg)
    # the oracle averages over its local frames and adds the trust term on every call:
    # re-weight to the global batch mean and keep the trust gradient on rank 0 only.
    _, tg = oracle.trust_region_penalty(d.atoms, d.anchor, np.float32(cfg.trust_delta), want_grad=True)
    trust = float(np.float32(cfg.lambda_feat)) * float(np.float32(cfg.lambda_trust)) * tg
    local = _flat(g, dp, da - trust) * (len(mine) / plan["global_batch"])
    if plan["add_trust"]:
        local[-da.size:] += trust.reshape(-1)
    t = torch.from_numpy(local.copy())
    dist.all_reduce(t)
    if rank == 0:
        _, (G, DP, DA) = oracle.total_objective(m, d, frames, intr, cfg)
        out.put((t.numpy(), _flat(G, DP, DA)))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2])
def test_sharded_gradients_equal_full_batch(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, ref = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_allclose(got, ref, rtol=1e-9, atol=1e-12)


KPART = 8


def _frame_partials(m, d, f, intr, cfg):
    """One frame's slot in the library's partials layout (latmap_loss_assemble), from the oracle's
    single-frame LossBreakdown (means -> the sums the device accumulates)."""
    loss, _ = oracle.total_objective(m, d, [f], intr, cfg, want_grad=False)
    h, w = f.depth.shape
    npx = h * w
    alpha = oracle.render(m, f.pose_rot, f.pose_trans, intr)["alpha"]
    valid = float(np.count_nonzero((f.depth.reshape(-1) > 0) & (alpha.reshape(-1) > 0.5)))
    nsup = float(loss["supervised_rows"])
    return np.array([loss["l_rgb"] * npx * 3, (1.0 - 2.0 * loss["l_ssim"]) * npx * 3,
                     loss["l_depth"] * valid, valid, loss["l_cos"] * nsup, loss["l_l2"] * nsup,
                     float(loss["zero_norm_flagged"]), nsup], np.float64), loss["l_trust"]


def _assembly_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_12314_b200 import api

    intr, m, d, frames = _problem()
    plan = rank_plan(len(frames), world, rank)
    cfg = oracle.Config()
    part = np.zeros(len(frames) * KPART + 16, np.float64)
    for i, gi in enumerate(plan["frames"]):
        slot = plan["slot_offset"] + i
        part[slot * KPART:(slot + 1) * KPART], trust = _frame_partials(m, d, frames[gi], intr, cfg)
        if plan["add_trust"]:
            part[len(frames) * KPART] = trust
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    if rank == 0:
        lcfg = api.default_config(**{k: float(getattr(cfg, k)) for k in (
            "lambda_cos", "lambda_l2", "lambda_trust", "trust_delta", "lambda_i1", "lambda_i2", "lambda_rgb",
            "lambda_depth", "lambda_feat")})
        got = api.assemble_loss(t.numpy(), intr.width, intr.height, lcfg)
        ref, _ = oracle.total_objective(m, d, frames, intr, cfg, want_grad=False)
        out.put((got, ref))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_partials_assemble_to_full_batch(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_assembly_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, ref = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust", "total"):
        assert got[k] == pytest.approx(ref[k], rel=1e-6, abs=1e-9), (k, got[k], ref[k])
    assert got["supervised_rows"] == ref["supervised_rows"]
