cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1940 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu94.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu94.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches94_cfg5.csv python bench.py --no-cpu --no-e2e --steps 1 --warmup 3 > gpurun_out/ncu94.log 2>&1
echo done
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b94_cfg5.json 2>/dev/null; timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b94_cfg3.json 2>/dev/null
