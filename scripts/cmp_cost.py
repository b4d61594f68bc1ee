"""Bit-compare the cached cost C (and one round's w, x) of two builds of libad2 on the same inputs:
    python scripts/cmp_cost.py libad2.so libad2_old.so [cfg N K]
A library argument may carry environment settings: libad2.so:AD2_COST_TILE4=1"""
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
ctx.init(t(b.offsets), t(b.supports), t(b.weights), t(b.labels), t(b.x0), t(b.w0), b.K, b.m, s.rho0, s.eps, s.rule)
C0 = ctx.member_matrices(ad2.COST)
ctx.step(10); ctx.update_support()
C1 = ctx.member_matrices(ad2.COST)
x, w = ctx.centroids()
np.savez(sys.argv[2], C0=np.concatenate([c.ravel() for c in C0]), C1=np.concatenate([c.ravel() for c in C1]),
         x=x, w=w, rho=ctx.rho())
print("variant", ctx.info()["variant"])
'''


def main():
    libs = sys.argv[1:3]
    cfg = sys.argv[3:6] or ["4", "3000", "5"]
    out = []
    for k, lib in enumerate(libs):
        f = f"/tmp/cmp_cost_{k}.npz"
        name, *kv = lib.split(":")
        env = dict(os.environ, AD2_LIB=os.path.join(ROOT, "paper_1510_00012_b200", name))
        env.update(dict(e.split("=", 1) for e in kv))
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT, f] + cfg, env=env, capture_output=True, text=True)
        print(lib, r.stdout.strip(), r.stderr.strip()[-500:])
        out.append(np.load(f))
    for key in ("C0", "C1", "x", "w", "rho"):
        a, b = out[0][key], out[1][key]
        print(key, a.shape, "bit-identical" if np.array_equal(a, b) else f"DIFFER max {np.abs(a - b).max()}")


if __name__ == "__main__":
    main()
