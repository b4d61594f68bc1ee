cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b87_cfg3a.json 2>/dev/null
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e --steps 10 > gpurun_out/b87_cfg3b.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches87_cfg3.csv python bench.py --workload 3 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu87.log 2>&1
echo done
