"""The tensor-core cost of the variant-2 iteration kernel (ad2_set_tc_cost): fp32
rounds with single-member 32-row passes and 4 < d <= 16 form x'_i . y'_j of the centred points
with tcgen05.mma kind::tf32 (hi/lo splits) in TMEM.  Held to the same north_star fp32 tolerances
against the fp64 oracle as the FFMA2 path (one iteration: Pi/w/x 1e-5 relative; full schedule:
objective 1e-3, w 1e-4 absolute, x 1e-3), at the BASELINE shapes, ragged shapes and on data far
from the origin (where the centring decides the accuracy of C = |x|^2 + |y|^2 - 2 x.y)."""
import dataclasses

import numpy as np
import pytest

import oracle
from paper_1510_00012_b200 import workloads as wl
from paper_1510_00012_b200 import ad2
from tests.harness import run_gpu, assert_hybrid
from tests.test_gpu_parity import compare_round

pytestmark = pytest.mark.gpu


def _tc_ctx(on):
    ctx = ad2.Context(0)
    ctx.set_tc_cost(on)
    return ctx


@pytest.mark.parametrize("cfg,N", [(3, 2000), (5, 3000)])
def test_tc_cost_in_use_and_matches_oracle(cfg, N):
    b = wl.make_config(cfg, N=N)
    ctx, _ = compare_round(b, T=1, tau=1, rtol_plan=1e-5, rtol_x=1e-5, atol_w=1e-6, ctx=_tc_ctx(1))
    assert ctx.info()["tc_cost"] == 1
    ctx, _ = compare_round(b, T=1, tau=1, rtol_plan=1e-5, rtol_x=1e-5, atol_w=1e-6, ctx=_tc_ctx(0))
    assert ctx.info()["tc_cost"] == 0


@pytest.mark.parametrize("cfg,N", [(3, 2000), (5, 3000)])
def test_tc_cost_full_schedule(cfg, N):
    b = wl.make_config(cfg, N=N)
    compare_round(b, T=b.sched.T, tau=b.sched.tau, rtol_plan=None, rtol_x=1e-3, atol_w=1e-4, rtol_obj=1e-3,
                  check_plans=False, ctx=_tc_ctx(1))


@pytest.mark.parametrize("m,mk,d", [(32, (1, 32), 16), (24, (3, 29), 9), (32, (4, 17), 5), (17, (1, 16), 12)])
def test_tc_cost_ragged_shapes(m, mk, d):
    """m < 32 (rows >= m padded), odd/even m_k from 1 to 32 (N = 16 and 32 MMAs), d < 16."""
    b = wl.make_random(400, m, d, K=3, mk_range=mk, seed=200 + m + d, dtype="f32", T=1, tau=1, spread=3.0)
    ctx, _ = compare_round(b, T=1, tau=1, rtol_plan=1e-5, rtol_x=1e-5, atol_w=1e-6, ctx=_tc_ctx(1))
    info = ctx.info()
    assert (info["variant"], info["mp"], info["tc_cost"]) == (2, 32, 1), info
    compare_round(b, T=9, tau=3, rtol_plan=None, rtol_x=1e-3, atol_w=1e-4, rtol_obj=1e-3, check_plans=False,
                  ctx=_tc_ctx(1))


def test_tc_cost_far_from_origin():
    """Every point and centroid shifted by +300 per coordinate: |x|^2 ~ 1.4e6 against costs ~ 30.
    The centred tensor-core products keep C at the data's scale (fp32 parity at 1e-5); C is
    translation invariant, so the oracle's plans are those of the unshifted instance."""
    b = wl.make_config(3, N=1500)
    sh = dataclasses.replace(b, supports=(b.supports + np.float32(300.0)).astype(b.supports.dtype),
                             x0=(b.x0 + np.float32(300.0)).astype(b.x0.dtype))
    compare_round(sh, T=1, tau=1, rtol_plan=1e-5, rtol_x=1e-5, atol_w=1e-6, ctx=_tc_ctx(1))


def test_tc_cost_equals_ffma_cost_path():
    """Both cost paths from the same start agree to the fp32 bar element by element (a step of 4:
    P1INIT, FUSED, FUSEDX; the support update; the objective)."""
    b = wl.make_config(5, N=2500)
    out = {}
    for on in (1, 0):
        ctx, rho, obj = run_gpu(b, T=4, tau=4, tc_cost=on)
        x, w = ctx.centroids()
        out[on] = (ctx.member_matrices(ad2.PI1), ctx.member_matrices(ad2.PI2), x, w, obj)
    p1a, p2a, xa, wa, oa = out[1]
    p1b, p2b, xb, wb, ob = out[0]
    assert_hybrid(np.concatenate([q.ravel() for q in p1a]), np.concatenate([q.ravel() for q in p1b]), 2e-5,
                  what="Pi1")
    assert_hybrid(np.concatenate([q.ravel() for q in p2a]), np.concatenate([q.ravel() for q in p2b]), 2e-5,
                  what="Pi2")
    assert np.abs(wa - wb).max() <= 1e-6
    assert_hybrid(xa, xb, 2e-5, floor=1.0, what="x")
    assert np.allclose(oa, ob, rtol=1e-5)
