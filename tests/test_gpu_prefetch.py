"""ad2_prefetch (host-batch pipelining): a round started from a prefetched host batch equals the
same round started from a plain host batch, bit for bit; a prefetch of other arrays is discarded
(the init copies its own); the batch buffers may be re-prefetched while a round is queued.  The
round itself is checked against the oracle by test_gpu_parity.py."""
import numpy as np
import pytest

import oracle
from paper_1510_00012_b200 import ad2, workloads as wl
from tests.harness import torch_cuda

pytestmark = pytest.mark.gpu


def host_arrays(b, torch):
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return {k: pin(getattr(b, k)) for k in ("offsets", "supports", "weights", "labels", "x0", "w0")}


def run_round(ctx, H, b, T=20, tau=10):
    ctx.init(H["offsets"], H["supports"], H["weights"], H["labels"], H["x0"], H["w0"], b.K, b.m,
             b.sched.rho0, b.sched.eps, b.sched.rule, mem="host", dtype=b.dtype)
    ad2.run_schedule(ctx, T, tau)
    obj = ctx.objective()
    x, w = ctx.centroids()
    return x, w, obj


@pytest.mark.parametrize("cfg,N,K", [(2, 3000, 4), (3, 800, 5)])
def test_prefetched_round_matches_plain_round(cfg, N, K):
    torch = torch_cuda()
    b = wl.make_config(cfg, N=N, K=K)
    H = host_arrays(b, torch)
    ref = ad2.Context(0)
    x0, w0, o0 = run_round(ref, H, b)
    ctx = ad2.Context(0)
    for rep in range(3):                               # prefetch -> init, repeatedly (buffer swaps)
        ctx.prefetch(H["offsets"], H["supports"], H["weights"], H["labels"], dtype=b.dtype)
        x, w, o = run_round(ctx, H, b)
        np.testing.assert_array_equal(x, x0)
        np.testing.assert_array_equal(w, w0)
        np.testing.assert_array_equal(o, o0)
    ctx.close()
    ref.close()


def test_prefetch_of_other_arrays_is_discarded():
    torch = torch_cuda()
    b1 = wl.make_config(2, N=1500, K=3)
    b2 = wl.make_config(2, N=1700, K=3)
    H1, H2 = host_arrays(b1, torch), host_arrays(b2, torch)
    ref = ad2.Context(0)
    x0, w0, o0 = run_round(ref, H2, b2)
    ctx = ad2.Context(0)
    ctx.prefetch(H1["offsets"], H1["supports"], H1["weights"], H1["labels"], dtype=b1.dtype)
    x, w, o = run_round(ctx, H2, b2)                   # different arrays: copies its own
    np.testing.assert_array_equal(x, x0)
    np.testing.assert_array_equal(o, o0)
    # the round matches the oracle cluster by cluster (objective, north_star fp32 tolerance)
    res, _ = oracle.run_bundle(b2, T=20, tau=10, want_state=False)
    for c, r in res.items():
        assert abs(o[c] - r.obj) <= 1e-3 * abs(r.obj) + 1e-9, (c, o[c], r.obj)
    ctx.close()
    ref.close()


def test_prefetch_while_a_round_is_queued():
    torch = torch_cuda()
    b = wl.make_config(3, N=600, K=4)
    H = host_arrays(b, torch)
    ref = ad2.Context(0)
    x0, _, o0 = run_round(ref, H, b)
    ctx = ad2.Context(0)
    ctx.init(H["offsets"], H["supports"], H["weights"], H["labels"], H["x0"], H["w0"], b.K, b.m,
             b.sched.rho0, b.sched.eps, b.sched.rule, mem="host", dtype=b.dtype)
    ad2.run_schedule(ctx, 20, 10)                      # queued, not synchronised
    ctx.prefetch(H["offsets"], H["supports"], H["weights"], H["labels"], dtype=b.dtype)
    o_first = ctx.objective()
    np.testing.assert_array_equal(o_first, o0)
    x, _, o = run_round(ctx, H, b)                     # consumes the prefetch
    np.testing.assert_array_equal(x, x0)
    np.testing.assert_array_equal(o, o0)
    ctx.close()
    ref.close()


def test_prefetch_argument_errors():
    b = wl.make_config(2, N=200, K=2)
    ctx = ad2.Context(0)
    assert ctx.L.ad2_prefetch(ctx.h, None, 0) == 1                 # AD2_ERR_ARG: no batch
    ctx.prefetch(b.offsets[:1], b.supports[:0], b.weights[:0], b.labels[:0], dtype=b.dtype)   # N = 0: no-op
    ctx.close()


def test_any_init_discards_a_pending_prefetch():
    """A prefetch not consumed by the next init is dropped: a later host init of the same (since
    rewritten) arrays copies them again instead of using the stale staged copy."""
    torch = torch_cuda()
    b = wl.make_config(2, N=1200, K=3)
    H = host_arrays(b, torch)
    ctx = ad2.Context(0)
    ctx.prefetch(H["offsets"], H["supports"], H["weights"], H["labels"], dtype=b.dtype)
    dev = {k: v.cuda() for k, v in H.items()}
    ctx.init(dev["offsets"], dev["supports"], dev["weights"], dev["labels"], dev["x0"], dev["w0"], b.K, b.m,
             b.sched.rho0, b.sched.eps, b.sched.rule, dtype=b.dtype)          # device init: discards it
    torch.cuda.synchronize()
    H["supports"].mul_(1.5)                                                       # same pointers, new data
    x, _, o = run_round(ctx, H, b)
    ref = ad2.Context(0)
    x0, _, o0 = run_round(ref, H, b)
    np.testing.assert_array_equal(x, x0)
    np.testing.assert_array_equal(o, o0)
    ctx.close()
    ref.close()
