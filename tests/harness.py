"""Shared test helpers: run the CUDA path (through the C ABI) and the oracle on the same bundle."""
from __future__ import annotations

import numpy as np

import oracle
from paper_1510_00012_b200 import workloads as wl


def torch_cuda():
    import torch
    assert torch.cuda.is_available()
    return torch


def to_dev(b: wl.Bundle, torch):
    dev = "cuda:0"
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    return dict(offsets=t(b.offsets), supports=t(b.supports), weights=t(b.weights), labels=t(b.labels),
                x0=t(b.x0), w0=t(b.w0))


def run_gpu(b: wl.Bundle, T=None, tau=None, rule=None, mem="device", nccl=False, ctx=None, warm_mask=None,
            x0=None, w0=None, profile=False, cost_mode=0, state_mode=0, eps=None, tc_cost=None):
    """Run one round of Alg. 4 on the GPU; returns (ctx, rho, objective)."""
    from paper_1510_00012_b200 import ad2
    torch = torch_cuda()
    s = b.sched
    T = s.T if T is None else T
    tau = s.tau if tau is None else tau
    rule = s.rule if rule is None else rule
    if ctx is None:
        ctx = ad2.Context(0)
        if nccl:
            ctx.attach_nccl(1, 0, ad2.nccl_unique_id())
    if profile:
        ctx.set_profiling(True)
    ctx.set_state_mode(state_mode)
    if tc_cost is not None:
        ctx.set_tc_cost(tc_cost)
    x0 = b.x0 if x0 is None else x0
    w0 = b.w0 if w0 is None else w0
    if mem == "device":
        a = to_dev(b, torch)
        a["x0"] = torch.from_numpy(np.ascontiguousarray(x0)).cuda()
        a["w0"] = torch.from_numpy(np.ascontiguousarray(w0)).cuda()
    else:
        a = dict(offsets=b.offsets, supports=b.supports, weights=b.weights, labels=b.labels,
                 x0=np.ascontiguousarray(x0), w0=np.ascontiguousarray(w0))
    rho = ctx.init(a["offsets"], a["supports"], a["weights"], a["labels"], a["x0"], a["w0"], b.K, b.m,
                   s.rho0, s.eps if eps is None else eps, rule, warm_mask=warm_mask, mem=mem, dtype=b.dtype, cost_mode=cost_mode)
    ad2.run_schedule(ctx, T, tau)
    obj = ctx.objective() if T > 0 else None
    torch.cuda.synchronize()
    return ctx, rho, obj


def hybrid_err(a, b, scale=None):
    """max |a-b| / (|b| + 1e-4*max|b|): relative with a floor for entries near eps."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    mx = np.abs(b).max() if b.size else 1.0
    return float((np.abs(a - b) / (np.abs(b) + (1e-4 if scale is None else scale) * mx)).max()) if b.size else 0.0


def assert_hybrid(a, b, rtol, floor=1e-4, what=""):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if b.size == 0:
        return
    tol = rtol * np.abs(b) + rtol * floor * np.abs(b).max()
    bad = np.abs(a - b) > tol
    if bad.any():
        idx = np.argmax(np.abs(a - b) - tol)
        raise AssertionError(f"{what}: {bad.sum()} / {b.size} entries off; worst a={a.ravel()[idx]!r} "
                             f"b={b.ravel()[idx]!r} tol={tol.ravel()[idx]!r}")
