"""ad2_set_profiling modes: 1 times every later step, 2 only the next step (the bench's live
kernel timing inside its timed region); profiling never changes the results."""
import numpy as np
import pytest

from paper_1510_00012_b200 import ad2, workloads as wl
from tests.harness import torch_cuda

pytestmark = pytest.mark.gpu


def _ctx(b, torch):
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ctx = ad2.Context(0)
    ctx.init(dev(b.offsets), dev(b.supports), dev(b.weights), dev(b.labels), dev(b.x0), dev(b.w0), b.K, b.m,
             b.sched.rho0, b.sched.eps, b.sched.rule, dtype=b.dtype)
    return ctx


def test_profile_next_step_only():
    torch = torch_cuda()
    b = wl.make_config(3, N=500, K=3)
    ctx = _ctx(b, torch)
    # variant-2 kernel: a step of n >= 2 iterations is n passes (the last one forms the x partials)
    extra = 0 if ctx.info()["variant"] == 2 else 1
    ctx.set_profiling(2)
    ctx.step(3)
    ms3, _ = ctx.prof_read()
    assert len(ms3) == 3 + extra and all(t > 0 for t in ms3)
    ctx.step(5)                                        # plain graph: the profiled step stays the last
    ms, _ = ctx.prof_read()
    assert len(ms) == 3 + extra
    ctx.set_profiling(1)
    ctx.step(5)
    ms5, _ = ctx.prof_read()
    assert len(ms5) == 5 + extra
    with pytest.raises(ad2.AD2Error):
        ctx.set_profiling(3)
    ctx.close()


def test_profiling_does_not_change_results():
    torch = torch_cuda()
    b = wl.make_config(3, N=500, K=3)
    out = []
    for mode in (0, 1, 2):
        ctx = _ctx(b, torch)
        ctx.set_profiling(mode)
        ad2.run_schedule(ctx, 20, 10)
        x, w = ctx.centroids()
        out.append((x, w, ctx.objective()))
        ctx.close()
    for x, w, o in out[1:]:
        np.testing.assert_array_equal(x, out[0][0])
        np.testing.assert_array_equal(w, out[0][1])
        np.testing.assert_array_equal(o, out[0][2])


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_cold_round_state_before_and_after_first_step(dtype):
    """A cold round with 32-row blocks forms Pi2^0 = w x w^(k) and Lambda = 0 inside its first pass
    (P1INIT); read back right after init they are materialised on demand and equal the product
    measure and zero, and the round's results match a round whose state was read
    (materialised) before its first step."""
    torch = torch_cuda()
    b = wl.make_config(3, N=300, K=3) if dtype == "f32" else \
        wl.make_random(300, 32, 4, K=3, mk_range=(3, 30), seed=5, dtype="f64")
    ctx = _ctx(b, torch)
    assert ctx.info()["variant"] == 2 and ctx.info()["mp"] == 32
    pi2 = ctx.member_matrices(ad2.PI2)
    lam = ctx.member_matrices(ad2.LAMBDA)
    w0 = np.asarray(b.w0, np.float64)
    for k in range(0, b.N, 37):
        c = int(b.labels[k])
        om = np.asarray(b.weights[b.offsets[k]:b.offsets[k + 1]], np.float64)
        om = om / om.sum()
        np.testing.assert_allclose(pi2[k], np.outer(w0[c], om), rtol=2e-6 if dtype == "f32" else 1e-14,
                                   atol=1e-12)
        assert not np.any(lam[k])
    ad2.run_schedule(ctx, 20, 10)
    x1, w1 = ctx.centroids()
    o1 = ctx.objective()
    ctx.close()
    ctx2 = _ctx(b, torch)                              # no read-back before the first step
    ad2.run_schedule(ctx2, 20, 10)
    x2, w2 = ctx2.centroids()
    np.testing.assert_array_equal(x1, x2)
    np.testing.assert_array_equal(w1, w2)
    np.testing.assert_array_equal(o1, ctx2.objective())
    ctx2.close()
