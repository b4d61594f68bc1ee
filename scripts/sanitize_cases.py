#!/usr/bin/env python
"""Small runs for scripts/sanitize.sh (compute-sanitizer): each case drives one kernel family
through the C ABI with shapes of configs 1/2 (a few hundred members) so the sanitizers finish."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_00012_b200 import ad2, workloads as wl  # noqa: E402


def round_(b, steps=((1, True), (3, True), (2, False), (1, False)), cost_mode=0):
    ctx = ad2.Context(0)
    s = b.sched
    ctx.init(b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0, b.K, b.m, s.rho0, s.eps, s.rule,
             mem="host", dtype=b.dtype, cost_mode=cost_mode)
    for n, upd in steps:
        ctx.step(n)
        if upd:
            ctx.update_support()
    ctx.objective()
    for which in (ad2.PI1, ad2.PI2, ad2.LAMBDA, ad2.COST):
        ctx.plans(which)
    x, w = ctx.centroids()
    warm = np.ones(b.N, np.uint8)
    warm[::2] = 0
    ctx.init(b.offsets, b.supports, b.weights, b.labels, x, w, b.K, b.m, s.rho0, s.eps, s.rule, warm_mask=warm,
             mem="host", dtype=b.dtype, cost_mode=cost_mode)
    ctx.step(4)
    ctx.update_support()
    ctx.objective()
    ctx.close()


def main(case):
    if case == "tma32":
        round_(wl.make_random(300, 32, 16, K=3, mk_range=(3, 32), seed=1, dtype="f32"))      # G = 1, pair layout
    elif case == "tma8":
        round_(wl.make_config(1))                                                           # fp64 MP 8
        round_(wl.make_random(300, 6, 2, K=2, mk_range=(1, 8), seed=2, dtype="f32"))         # G = 4
    elif case == "tma16_2ch":
        round_(wl.make_random(300, 12, 3, K=2, mk_range=(10, 32), seed=3, dtype="f32"))      # MP 16, two chunks
    elif case == "f64":
        round_(wl.make_random(200, 24, 5, K=2, mk_range=(3, 29), seed=4, dtype="f64"))
        round_(wl.make_random(100, 40, 3, K=2, mk_range=(3, 20), seed=5, dtype="f64"))       # generic kernel
    elif case == "wide64":
        round_(wl.make_config(4, N=150, K=3))                                               # warp pair, d = 64
    elif case == "wide32":
        round_(wl.make_random(200, 20, 24, K=2, mk_range=(3, 50), seed=6, dtype="f32"))      # warp per member
        round_(wl.make_random(60, 100, 5, K=2, mk_range=(20, 64), seed=7, dtype="f32"))      # warp quad
    elif case == "tc":
        round_(wl.make_config(4, N=150, K=3), cost_mode=1)                                  # tcgen05 cost build
    elif case == "assign":
        b = wl.make_config(3, N=200, K=6)
        ctx = ad2.Context(0)
        ctx.assign(b.offsets, b.supports, b.weights, b.x0, b.w0, mem="host", dtype=b.dtype)
        picks = np.arange(b.K, dtype=np.int64) * 7
        ctx.merge_init(b.offsets, b.supports, b.weights, picks, b.K, b.m, mem="host")
        ctx.close()
    elif case == "group":
        g = ad2.Group(f"/ad2s_{os.getpid()}", 1, 0)
        ctx = ad2.Context(0)
        ctx.attach_group(g)
        b = wl.make_random(200, 16, 3, K=2, mk_range=(2, 14), seed=8, dtype="f64")
        ctx.init(b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0, b.K, b.m, mem="host", dtype="f64")
        ad2.run_schedule(ctx, 6, 3)
        ctx.objective()
        ctx.close()
        g.close()
    print(f"case {case} ok")


if __name__ == "__main__":
    main(sys.argv[1])
