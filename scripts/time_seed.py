"""Time the initial partition on the device (ad2_kmeanspp + ad2_label_nearest + ad2_pick_members +
ad2_merge_init) at a config's full size, beside the harness's host numpy version (workloads).

    python scripts/time_seed.py --cfg 5
"""
import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_00012_b200 import ad2, workloads as wl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    import torch
    b = wl.make_config(a.cfg)
    K = b.K
    ns = max(K, int(round(0.1 * b.N)))
    rng = np.random.default_rng(1)
    sample = rng.choice(b.N, size=ns, replace=False)
    u, up = rng.uniform(size=K), rng.uniform(size=K)
    t = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    off, Y, W = t(b.offsets), t(b.supports), t(b.weights)
    ctx = ad2.Context(0)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cen = ctx.kmeanspp(off, Y, W, sample, u, a.iters, dtype=b.dtype)
        t1 = time.perf_counter()
        lab, cen2 = ctx.label_nearest(off, Y, W, cen, dtype=b.dtype)
        t2 = time.perf_counter()
        pick = ctx.pick_members(off, Y, W, t(lab), b.m, up, dtype=b.dtype)
        t3 = time.perf_counter()
        x0, w0 = ctx.merge_init(off, Y, W, pick, K, b.m, dtype=b.dtype)
        t4 = time.perf_counter()
        print(f"cfg{a.cfg} N={b.N} ns={ns} K={K} d={b.d} rep {rep}: kmeanspp {1e3*(t1-t0):.1f} ms, "
              f"label_nearest {1e3*(t2-t1):.1f} ms, pick {1e3*(t3-t2):.1f} ms, merge_init {1e3*(t4-t3):.1f} ms, "
              f"sizes min/max {np.bincount(lab, minlength=K).min()}/{np.bincount(lab, minlength=K).max()}",
              flush=True)
    mu = wl.member_means(b)
    t0 = time.perf_counter()
    wl.kmeanspp(mu[sample], K, np.random.default_rng(2), a.iters)
    print(f"host harness kmeanspp (numpy, same sample size): {1e3*(time.perf_counter()-t0):.0f} ms", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
