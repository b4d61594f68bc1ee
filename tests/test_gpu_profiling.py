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
    ctx.set_profiling(2)
    ctx.step(3)
    ms3, _ = ctx.prof_read()
    assert len(ms3) == 4 and all(t > 0 for t in ms3)
    ctx.step(5)                                        # plain graph: the profiled step stays the last
    ms, _ = ctx.prof_read()
    assert len(ms) == 4
    ctx.set_profiling(1)
    ctx.step(5)
    ms5, _ = ctx.prof_read()
    assert len(ms5) == 6
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
