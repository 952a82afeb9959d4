"""The keyframe-sharded step through the LIBRARY on one GPU: two
sessions stand in for two ranks, each holding half of the 8-frame window with
set_batch(global_batch=8, add_trust=(rank == 0), slot_offset=first frame). Summing their gradient
and loss-partial buffers (what latmap_session_allreduce does across ranks) must reproduce a
full-batch session: the batch mean uses the GLOBAL batch (proj/src/objective.cpp:77) and the
trust-region term enters once (objective.cpp:176-185). No rank waits on another's kernels here:
the sessions run one after the other and the sum is a plain device add."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_12314_b200 import api, synthetic  # noqa: E402
from paper_2602_12314_b200.sharding import rank_plan  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return api.Context(0)


def gpu_render(ctx):
    def fn(m, q, t, intr):
        out = api.render(ctx, api.GaussianMap.from_numpy(m), api.make_pose(q, t),
                         api.make_intrinsics(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
        return out.color.cpu().numpy(), out.depth.cpu().numpy(), out.alpha.cpu().numpy()
    return fn


def session(ctx, w, frames, precision):
    cfg = api.default_config(**w.lambdas)
    cfg.decoder_precision = precision
    intr = api.make_intrinsics(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height)
    s = api.Session(ctx, cfg, w.map.n, w.map.features.shape[1], w.atoms.shape[0], w.atoms.shape[1], intr)
    s.set_map(w.map)
    s.set_dictionary(w.atoms, w.anchor, w.proj)
    s.set_frames(frames)
    return s, cfg


@pytest.mark.parametrize("world,precision", [(2, 1), (4, 1), (2, 0)])
def test_sharded_sessions_sum_to_full_batch(ctx, world, precision):
    w = synthetic.make_workload(2, gpu_render(ctx), scale=0.25)
    nf = len(w.frames)
    full, cfg = session(ctx, w, w.frames, precision)
    full.set_batch(nf)
    ref_loss = full.objective(want_grad=True)
    ref_g = full.grad_buffer().clone()
    ref_p = full.loss_buffer().clone()

    g_sum = torch.zeros_like(ref_g)
    p_sum = torch.zeros_like(ref_p)
    for r in range(world):
        plan = rank_plan(nf, world, r)
        s, _ = session(ctx, w, [w.frames[i] for i in plan["frames"]], precision)
        s.set_batch(plan["global_batch"], add_trust=plan["add_trust"], slot_offset=plan["slot_offset"])
        s.objective(want_grad=True, read=False)
        g_sum += s.grad_buffer()
        p_sum += s.loss_buffer()
        del s
    torch.cuda.synchronize()
    # gradients: equal up to the float-atomic order of the per-splat / dictionary sums
    rel = float(torch.linalg.norm(g_sum - ref_g) / torch.linalg.norm(ref_g))
    assert rel < 1e-5, rel
    # loss partials: per-frame slots are disjoint (slot_offset), the trust slot comes from rank 0 only
    np.testing.assert_allclose(p_sum.cpu().numpy(), ref_p.cpu().numpy(), rtol=1e-9, atol=1e-12)
    # the library's host assembly of the summed partials == the full session's LossBreakdown
    got = api.assemble_loss(p_sum.cpu().numpy(), w.intr.width, w.intr.height, cfg)
    for k in ("l_rgb", "l_ssim", "l_depth", "l_cos", "l_l2", "l_trust", "total"):
        assert got[k] == pytest.approx(ref_loss[k], rel=1e-6, abs=1e-9), (k, got[k], ref_loss[k])
    assert got["supervised_rows"] == ref_loss["supervised_rows"]


def test_sharded_step_applies_identical_adam(ctx):
    """sharded_step with a summing exchange: two 'ranks' (4 + 4 frames) exchange through device
    buffers; after the step both hold the map a full-batch step produces (same Adam input up to
    the atomic order of the sums, so the same parameters to float noise)."""
    w = synthetic.make_workload(2, gpu_render(ctx), scale=0.25)
    nf = len(w.frames)
    full, _ = session(ctx, w, w.frames, 1)
    full.set_batch(nf)
    full.step(read=True)
    ref_params = full.export_rows().clone()

    ranks = []
    for r in range(2):
        plan = rank_plan(nf, 2, r)
        s, _ = session(ctx, w, [w.frames[i] for i in plan["frames"]], 1)
        s.set_batch(plan["global_batch"], add_trust=plan["add_trust"], slot_offset=plan["slot_offset"])
        ranks.append(s)
    # objective on both, then the exchange (sum into each), then apply on both
    for s in ranks:
        s.objective(want_grad=True, read=False)
    g = ranks[0].grad_buffer() + ranks[1].grad_buffer()
    p = ranks[0].loss_buffer() + ranks[1].loss_buffer()
    for s in ranks:
        s.grad_buffer().copy_(g)
        s.loss_buffer().copy_(p)
        s.apply()
        assert not s.check_overflow()
        assert s.overflow_steps() == 0
    a, b = (s.export_rows() for s in ranks)
    assert torch.equal(a, b)  # identical Adam input -> identical parameters on every rank
    rel = float(torch.linalg.norm(a - ref_params) / torch.linalg.norm(ref_params))
    assert rel < 1e-5, rel


@pytest.mark.parametrize("inject_nan", [False, True])
def test_zero1_sharded_adam_equals_replicated(ctx, inject_nan):
    """The ZeRO-1 step (latmap_session_exchange_sharded's pieces, NCCL replaced by device adds and
    copies on one GPU): reduce-scatter -> shard check -> partials all-reduce (block skip flags
    OR-ed) -> Adam on each rank's shard -> all-gather. Bit-identical to every rank applying the
    replicated Adam to the same summed gradients, including a whole-block skip for a non-finite
    gradient found in only one rank's shard (adam.hpp:65-68)."""
    w = synthetic.make_workload(2, gpu_render(ctx), scale=0.25)
    nf = len(w.frames)
    ranks = []
    for r in range(2):
        plan = rank_plan(nf, 2, r)
        s, _ = session(ctx, w, [w.frames[i] for i in plan["frames"]], 1)
        s.set_batch(plan["global_batch"], add_trust=plan["add_trust"], slot_offset=plan["slot_offset"])
        ranks.append(s)
    rep, _ = session(ctx, w, [w.frames[i] for i in rank_plan(nf, 2, 0)["frames"]], 1)
    rep.set_batch(nf, add_trust=True, slot_offset=0)
    for s in ranks + [rep]:
        s.objective(want_grad=True, read=False)
    g = ranks[0].grad_buffer() + ranks[1].grad_buffer()
    p = ranks[0].loss_buffer() + ranks[1].loss_buffer()
    total = g.numel()
    (b0, e0), (b1, e1) = ranks[0].shard_range(2, 0), ranks[1].shard_range(2, 1)
    assert b0 == 0 and e0 == b1 and e1 == total and b1 % 4 == 0
    bad_block = None
    if inject_nan:  # a non-finite gradient in rank 1's shard only
        bad_block = next(nm for nm, (o, n) in ranks[1].grad_blocks().items() if o <= b1 + 1 < o + n)
        g[b1 + 1] = float("nan")
    init = ranks[0].params_buffer().clone()
    # replicated: every rank applies Adam to the all-reduced gradients
    rep.grad_buffer().copy_(g)
    rep.loss_buffer().copy_(p)
    rep.apply()
    # sharded: reduce-scatter (each rank keeps the summed gradients of its shard) ...
    tail = p.numel() - 16
    for s in ranks:
        s.grad_buffer().copy_(g)
        s.loss_buffer().copy_(p)
    ranks[0].shard_check(b0, e0)
    ranks[1].shard_check(b1, e1)
    # ... partials all-reduce: the per-block skip flags of the two shards OR-ed ...
    flags = ranks[0].loss_buffer()[tail + 2:tail + 10] + ranks[1].loss_buffer()[tail + 2:tail + 10]
    assert bool(flags.any().item()) == inject_nan
    for s in ranks:
        s.loss_buffer()[tail + 2:tail + 10] = flags
    # ... Adam on each shard, then all-gather of the parameters
    ranks[0].apply_range(b0, e0)
    ranks[1].apply_range(b1, e1)
    p0, p1 = ranks[0].params_buffer(), ranks[1].params_buffer()
    p0[b1:e1] = p1[b1:e1]
    p1[b0:e0] = p0[b0:e0]
    torch.cuda.synchronize()
    ref = rep.params_buffer()
    assert torch.equal(p0, ref) and torch.equal(p1, ref)
    if inject_nan:  # that whole block was skipped on both ranks (also the part in rank 0's shard)
        o, n = ranks[0].grad_blocks()[bad_block]
        assert torch.equal(p0[o:o + n], init[o:o + n]) and o < b1, bad_block
    else:
        assert not torch.equal(p0, init)
