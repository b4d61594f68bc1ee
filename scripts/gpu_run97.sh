cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_symbolic.py -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu97.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu97.log
timeout 900 python bench.py --workload 4 --no-cpu --no-e2e > gpurun_out/b97_cfg4.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cost_tile" -c 3 python scripts/prof_round.py --cfg 4 > gpurun_out/ncu97.log 2>&1
echo done
