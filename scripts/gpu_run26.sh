cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for p in 1 2 4 8; do AD2_PASSES=$p timeout 300 python bench.py --workload 2 --no-cpu --no-e2e --steps 5 > gpurun_out/b26_cfg2_p$p.json 2>/dev/null; done
for p in 8 16 32 64; do AD2_PASSES=$p timeout 600 python bench.py --workload 3 --no-cpu --no-e2e --steps 3 > gpurun_out/b26_cfg3_p$p.json 2>/dev/null; done
echo done
