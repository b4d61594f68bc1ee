cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu32.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu32.log
timeout 900 python bench.py --no-cpu --no-e2e --steps 3 > gpurun_out/b32_cfg5.json 2>/dev/null
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e --steps 3 > gpurun_out/b32_cfg3.json 2>/dev/null
timeout 900 python bench.py --workload 4 --no-cpu --no-e2e --steps 2 > gpurun_out/b32_cfg4.json 2>/dev/null
timeout 900 python bench.py --workload 2 --no-cpu --no-e2e --steps 5 > gpurun_out/b32_cfg2.json 2>/dev/null
echo done
