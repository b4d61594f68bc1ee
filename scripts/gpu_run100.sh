cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for p in 8 4 16 32; do AD2_PASSES=$p timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b100_p$p.json 2>/dev/null; done
for p in 8 4 16; do AD2_PASSES=$p timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b100_c3_p$p.json 2>/dev/null; done
echo done
