cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu36.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu36.log
timeout 900 python bench.py --workload 4 --no-cpu --no-e2e --steps 2 > gpurun_out/b36_cfg4.json 2>/dev/null
echo done
