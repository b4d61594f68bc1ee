cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench29_cfg5.json 2> gpurun_out/bench29_cfg5.err
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/bench29_cfg3.json 2>/dev/null
timeout 900 python bench.py --workload 4 --no-cpu --no-e2e > gpurun_out/bench29_cfg4.json 2>/dev/null
timeout 900 python bench.py --workload 2 --no-cpu --no-e2e > gpurun_out/bench29_cfg2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches29_cfg5.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu29_launch.log 2>&1
echo done
