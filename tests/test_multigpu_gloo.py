"""The N>1 keyframe-sharded path on CPU: 2 ranks over gloo. Each rank evaluates its shard of
the window with the global batch mean (the CPU oracle stands in for the device step, which
needs a GPU), the gradient buffers are summed with all_reduce, and the result must equal the
full-batch gradient of total_objective (objective.cpp:67-194)."""
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
