cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu33.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu33.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/b33_cfg5.json 2>/dev/null
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e --steps 3 > gpurun_out/b33_cfg3.json 2>/dev/null
echo done
