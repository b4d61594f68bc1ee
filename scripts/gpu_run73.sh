cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_symbolic.py tests/test_gpu_prefetch.py -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu73.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu73.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b73_cfg5.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_cost_member" -c 4 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu73.log 2>&1
echo done
