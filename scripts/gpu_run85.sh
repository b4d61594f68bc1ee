cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/b85_cfg5.json 2>gpurun_out/b85_cfg5.err
timeout 900 python bench.py --workload 3 > gpurun_out/b85_cfg3.json 2>/dev/null
timeout 900 python bench.py --workload 4 > gpurun_out/b85_cfg4.json 2>/dev/null
timeout 900 python bench.py --workload 2 > gpurun_out/b85_cfg2.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches85_cfg5.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu85.log 2>&1
echo done
