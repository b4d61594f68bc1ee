cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 1200 -p no:cacheprovider > gpurun_out/pytest_gpu72.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu72.log
timeout 900 python bench.py --no-cpu --no-e2e > gpurun_out/b72_cfg5.json 2>/dev/null
timeout 900 python bench.py --workload 3 --no-cpu --no-e2e > gpurun_out/b72_cfg3.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_badmm_tma" -s 3 -c 1 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu72.log 2>&1
echo done
