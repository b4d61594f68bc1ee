"""Wall-clock split of a round (init / schedule / objective) on a config (diagnostic)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_00012_b200 import ad2, workloads as wl  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
b = wl.make_config(cfg)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = [dev(a) for a in (b.offsets, b.supports, b.weights, b.labels, b.x0, b.w0)]
ctx = ad2.Context(0, torch.cuda.current_stream().cuda_stream)
s = b.sched
for r in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ctx.init(*D, b.K, b.m, s.rho0, s.eps, s.rule, dtype=b.dtype)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    ts = []
    done = 0
    while done < s.T:
        a = time.perf_counter(); ctx.step(s.tau); b1 = time.perf_counter(); ctx.update_support(); c = time.perf_counter()
        ts.append((b1 - a, c - b1)); done += s.tau
    torch.cuda.synchronize(); t2 = time.perf_counter()
    ctx.objective(); t3 = time.perf_counter()
    print(f"round {r}: init {1e3*(t1-t0):.2f} ms, schedule {1e3*(t2-t1):.2f} ms (host step/update calls: "
          + ", ".join(f"{1e3*x:.2f}/{1e3*y:.2f}" for x, y in ts) + f"), objective {1e3*(t3-t2):.2f} ms", flush=True)
