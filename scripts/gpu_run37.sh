cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_assign.py tests/test_gpu_symbolic.py -m gpu -q -x --timeout 500 -p no:cacheprovider > gpurun_out/pytest_gpu37.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu37.log
timeout 300 python scripts/time_assign.py --cfg 3 > gpurun_out/ta37.log 2>&1
timeout 300 python scripts/time_assign.py --cfg 5 --N 400000 >> gpurun_out/ta37.log 2>&1
timeout 300 python scripts/time_assign.py --cfg 4 --N 100000 >> gpurun_out/ta37.log 2>&1
echo done
