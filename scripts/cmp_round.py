"""Bit-compare one round (init + T/tau x (step, update) + objective) of two builds of libad2 on the
same inputs: Pi1, Lambda, x, w, rho, objective.
    python scripts/cmp_round.py libad2.so libad2_old.so [cfg N K]"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1510_00012_b200 import ad2, workloads as wl
cfg, N, K = int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
b = wl.make_config(cfg, N=N, K=K)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
ctx = ad2.Context(0)
s = b.sched
rho = ctx.init(t(b.offsets), t(b.supports), t(b.weights), t(b.labels), t(b.x0), t(b.w0), b.K, b.m, s.rho0, s.eps, s.rule)
ad2.run_schedule(ctx, 20, 10)
obj = ctx.objective()
x, w = ctx.centroids()
P = ctx.member_matrices(ad2.PI1)
np.savez(sys.argv[2], P=np.concatenate([p.ravel() for p in P]), x=x, w=w, rho=rho, obj=obj)
'''


def main():
    libs = sys.argv[1:3]
    cfg = sys.argv[3:6] or ["5", "20000", "16"]
    out = []
    for k, lib in enumerate(libs):
        f = f"/tmp/cmp_round_{k}.npz"
        env = dict(os.environ, AD2_LIB=os.path.join(ROOT, "paper_1510_00012_b200", lib))
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT, f] + cfg, env=env, capture_output=True, text=True)
        print(lib, r.stdout.strip(), r.stderr.strip()[-300:])
        out.append(np.load(f))
    for key in ("P", "x", "w", "rho", "obj"):
        a, b = out[0][key], out[1][key]
        print(key, a.shape, "bit-identical" if np.array_equal(a, b) else f"DIFFER max {np.abs(a - b).max()}")


if __name__ == "__main__":
    main()
