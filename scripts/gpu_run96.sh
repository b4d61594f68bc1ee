cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_symbolic.py tests/test_gpu_prefetch.py -m gpu -q -x -p no:cacheprovider -k "not full" > gpurun_out/pytest_gpu96.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu96.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_gather" -c 2 python scripts/prof_round.py --cfg 5 > gpurun_out/ncu96.log 2>&1
echo done
