cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_profiling.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu78.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu78.log
for c in 5 3 2; do timeout 900 python bench.py --workload $c --no-cpu > gpurun_out/b78_cfg$c.json 2>/dev/null; done
echo done
