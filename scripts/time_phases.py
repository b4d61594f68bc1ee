"""Wall-clock breakdown of one round through the C ABI (init / steps / support updates / objective).
Not a bench number: a diagnostic for where a round's time goes."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_00012_b200 import ad2, workloads as wl  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--rounds", type=int, default=3)
args = ap.parse_args()
t = time.time()
b = wl.make_config(args.cfg)
print(f"gen {time.time() - t:.1f}s", flush=True)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = [dev(a) for a in (b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0)]
ctx = ad2.Context(0, torch.cuda.current_stream().cuda_stream)
s = b.sched


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for r in range(args.rounds):
    t0 = tick()
    ctx.init(*D, b.K, b.m, s.rho0, s.eps, s.rule, dtype=b.dtype)
    t1 = tick()
    st, up = 0.0, 0.0
    for e in range(s.T // s.tau):
        a0 = tick()
        ctx.step(s.tau)
        a1 = tick()
        ctx.update_support()
        a2 = tick()
        st += a1 - a0
        up += a2 - a1
    t2 = tick()
    obj = ctx.objective()
    t3 = tick()
    print(f"round {r}: init {1e3 * (t1 - t0):.1f} ms, steps {1e3 * st:.1f} ms, updates {1e3 * up:.1f} ms, "
          f"objective {1e3 * (t3 - t2):.1f} ms, total {1e3 * (t3 - t0):.1f} ms", flush=True)
