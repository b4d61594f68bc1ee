cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b90_cfg5.json 2>/dev/null
for i in 1 2 3; do timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b90_cfg3_$i.json 2>gpurun_out/b90_cfg3_$i.err; done
echo done
