cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python bench.py --workload 2 --no-cpu --no-e2e > gpurun_out/b58_cfg2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches58_cfg2.csv python bench.py --workload 2 --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu58.log 2>&1
echo done
