"""The library's NCCL communicator (latmap_comm_*) on one GPU: a one-rank
communicator's sum all-reduce is the identity, and the session exchange
(latmap_session_allreduce) leaves the step's gradients and loss partials unchanged between
objective and apply. Multi-rank behaviour is NCCL's own sum over the same buffers."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2602_12314_b200 import _capi, api  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return api.Context(0)


def test_one_rank_allreduce_is_identity(ctx):
    uid = api.Comm.unique_id(ctx)
    assert len(uid) == 128
    comm = api.Comm(ctx, 1, 0, uid)
    for dt in (torch.float32, torch.float64):
        t = torch.randn(100003, device="cuda", dtype=dt)
        ref = t.clone()
        comm.allreduce(t)
        ctx.sync()
        assert torch.equal(t, ref)
    with pytest.raises(_capi.InvalidArgument):
        comm.allreduce(torch.zeros(4, device="cuda", dtype=torch.int32))
    with pytest.raises(_capi.InvalidArgument):
        api.Comm(ctx, 1, 0, b"short")


def test_session_allreduce_between_objective_and_apply(ctx):
    from paper_2602_12314_b200 import synthetic
    import oracle

    def orender(m, q, t, intr):
        om = oracle.GaussianMap(*[np.ascontiguousarray(getattr(m, f), np.float32) for f in oracle.FIELDS])
        out = oracle.render(om, q, t, oracle.make_intr(intr.fx, intr.fy, intr.cx, intr.cy, intr.width, intr.height))
        return out["color"], out["depth"], out["alpha"]

    w = synthetic.make_workload(0, orender)
    intr = api.make_intrinsics(w.intr.fx, w.intr.fy, w.intr.cx, w.intr.cy, w.intr.width, w.intr.height)
    s = api.Session(ctx, api.default_config(**w.lambdas), w.map.n, w.map.features.shape[1], w.atoms.shape[0],
                    w.atoms.shape[1], intr)
    s.set_map(w.map)
    s.set_dictionary(w.atoms, w.anchor, w.proj)
    s.set_frames(w.frames)
    comm = api.Comm(ctx, 1, 0, api.Comm.unique_id(ctx))
    s.objective(want_grad=True, read=False)
    ctx.sync()
    g0, p0 = s.grad_buffer().clone(), s.loss_buffer().clone()
    comm.session_allreduce(s)
    ctx.sync()
    assert torch.equal(s.grad_buffer(), g0) and torch.equal(s.loss_buffer(), p0)
    s.apply()
    loss = s.read_loss()
    assert np.isfinite(loss["total"])
